"""CPU (gloo, world_size 2): the N>1 path of bench.py runs one replica per
rank and reports rank 0's line with the step time maxed over ranks.  This
test drives that host logic with two gloo ranks on 127.0.0.1: every rank
factorizes the same seeded input with the CPU oracle, the results must be
bit-identical across ranks (the reference's worker-count determinism,
SPEC.md:161/:545, in replica form), and the max-over-ranks reduction used for
the timing behaves as bench.py assumes."""
import hashlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _digest(f):
    h = hashlib.sha256()
    for st in f.stages:
        for a in (st.cluster_offsets, st.members, st.rot_indices, st.rot_matrices, st.elim_index, st.elim_diagonal):
            h.update(np.ascontiguousarray(a).tobytes())
    h.update(np.ascontiguousarray(f.core).tobytes())
    h.update(np.float64(f.residual_sq).tobytes())
    return h.digest()


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import cases
    import oracles

    inp, params, part = cases.build("rmat10_m8")
    f = oracles.factorize("oracle", inp, params, part)
    d = torch.tensor(list(_digest(f)), dtype=torch.uint8)
    gathered = [torch.zeros_like(d) for _ in range(world)]
    dist.all_gather(gathered, d)
    same = all(torch.equal(g, gathered[0]) for g in gathered)
    t = torch.tensor([10.0 * (rank + 1)], dtype=torch.float64)  # stand-in step times
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    rots = sum(len(s.rot_indices) for s in f.stages)
    if rank == 0:
        out.put((same, float(t.item()), rots))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_gloo_ranks_replicas_identical():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    same, tmax, rots = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    assert same, "replicas differ across ranks"
    assert tmax == 20.0  # max over ranks
    assert rots > 0
