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


def shard_ranges_py(sizes, nnz, world, apply_weight=64):
    """Restatement of shard.cu shard_ranges: contiguous split of the clusters
    by the cost prefix c^2 + 64 nnz, each boundary on the side nearer r/W."""
    m = len(sizes)
    pre = [0.0]
    for u in range(m):
        pre.append(pre[-1] + float(sizes[u]) * float(sizes[u]) + apply_weight * float(nnz[u] if nnz is not None else 0))
    lo = [0] + [m] * world
    u = 0
    for r in range(1, world):
        target = pre[m] * r / world
        while u < m and pre[u + 1] <= target:
            u += 1
        b = u + 1 if (u < m and target - pre[u] > pre[u + 1] - target) else u
        lo[r] = max(b, lo[r - 1])
    lo[world] = m
    return lo


def _shard_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from paper_1507_04396_b200 import api

    # the communicator bootstrap: rank 0's NCCL id reaches every rank intact
    box = [api.Communicator.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    ids = [None] * world
    dist.all_gather_object(ids, box[0])
    # every rank derives the same cluster split from the same stage partition
    rng = np.random.default_rng(7)
    sizes = rng.integers(10, 5000, size=517)
    nnz = sizes * rng.integers(2, 40, size=517)
    splits = {}
    for w in (2, 3, 8):
        splits[w] = api.shard_ranges(sizes, nnz, w).tolist()
    all_splits = [None] * world
    dist.all_gather_object(all_splits, splits)
    if rank == 0:
        out.put((ids, all_splits, sizes.tolist(), nnz.tolist()))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_gloo_ranks_shard_plan():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ids, all_splits, sizes, nnz = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    assert len(ids[0]) == 128 and ids[0] == ids[1]
    assert all_splits[0] == all_splits[1]
    for w, lo in all_splits[0].items():
        assert lo == shard_ranges_py(sizes, nnz, w)
        assert lo[0] == 0 and lo[-1] == len(sizes) and all(a <= b for a, b in zip(lo, lo[1:]))
        cost = [s * s + 64 * z for s, z in zip(sizes, nnz)]
        share = [sum(cost[lo[r]:lo[r + 1]]) for r in range(w)]
        assert max(share) <= sum(cost) / w + max(cost)  # balanced to one cluster


def test_shard_ranges_edges():
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1507_04396_b200 import api

    assert api.shard_ranges([], None, 3).tolist() == [0, 0, 0, 0]
    assert api.shard_ranges([5], None, 4).tolist() == shard_ranges_py([5], None, 4)
    assert api.shard_ranges([100] * 10, None, 4).tolist() == [0, 2, 5, 7, 10]
    assert api.shard_ranges([3, 1, 4, 1, 5, 9, 2, 6], [1] * 8, 1).tolist() == [0, 8]


def _a2a_worker(rank, world, port, out):
    """The owned-column exchange of shard.cu redistribute(), message for
    message, over gloo: every rank holds a full-width CSC slab of the columns
    it owned before the reblock; the product's shard_ranges (C-ABI host code)
    assigns the new clusters; each rank sends, per destination, the column
    lengths of the destination's range and the entries of those columns
    (counts exchanged first, as the NCCL path does), and rebuilds its new
    slab from the per-source lengths (every column comes from one source)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from paper_1507_04396_b200 import api

    rng = np.random.default_rng(11)
    N = 300
    dense = (rng.random((N, N)) < 0.05) * rng.standard_normal((N, N))
    old_cut = [0, 137, N]  # the old ownership (column ranges)
    ptr = np.zeros(N + 1, np.int64)
    rows, vals = [], []
    for c in range(N):
        if old_cut[rank] <= c < old_cut[rank + 1]:
            nz = np.nonzero(dense[:, c])[0]
            rows += nz.tolist()
            vals += dense[nz, c].tolist()
        ptr[c + 1] = len(rows)
    rows, vals = np.array(rows, np.int32), np.array(vals)
    sizes = rng.integers(5, 40, size=12)
    sizes[-1] = N - sizes[:-1].sum() if sizes[:-1].sum() < N else 1
    off = np.concatenate([[0], np.cumsum(sizes)])
    off[-1] = N
    nnz = [int(np.count_nonzero(dense[:, off[u]:off[u + 1]])) for u in range(len(sizes))]
    lo = api.shard_ranges(sizes, nnz, world).tolist()
    dest = [int(off[min(x, len(sizes))]) for x in lo]
    at = [int(ptr[d]) for d in dest]
    # counts[s][d]: all-gathered
    mine = torch.tensor([at[d + 1] - at[d] for d in range(world)], dtype=torch.int64)
    allc = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allc, mine)
    reqs, recv_len, recv_row, recv_val = [], {}, {}, {}
    for d in range(world):
        if d == rank:
            continue
        lens = torch.tensor(np.diff(ptr[dest[d]:dest[d + 1] + 1]), dtype=torch.int64)
        reqs.append(dist.isend(lens, d))
        reqs.append(dist.isend(torch.tensor(rows[at[d]:at[d + 1]]), d))
        reqs.append(dist.isend(torch.tensor(vals[at[d]:at[d + 1]]), d))
    n = dest[rank + 1] - dest[rank]
    for src in range(world):
        if src == rank:
            continue
        k = int(allc[src][rank])
        recv_len[src] = torch.zeros(n, dtype=torch.int64)
        recv_row[src] = torch.zeros(k, dtype=torch.int32)
        recv_val[src] = torch.zeros(k, dtype=torch.float64)
        dist.recv(recv_len[src], src)
        dist.recv(recv_row[src], src)
        dist.recv(recv_val[src], src)
    for r in reqs:
        r.wait()
    recv_len[rank] = torch.tensor(np.diff(ptr[dest[rank]:dest[rank + 1] + 1]), dtype=torch.int64)
    recv_row[rank] = torch.tensor(rows[at[rank]:at[rank + 1]])
    recv_val[rank] = torch.tensor(vals[at[rank]:at[rank + 1]])
    # the new slab: lengths summed over sources, entries copied per source
    new = np.zeros((N, n))
    total = sum(recv_len[s] for s in range(world))
    assert all(((recv_len[s] > 0).int() + (recv_len[t] > 0).int() <= 1).all()
               for s in range(world) for t in range(world) if s < t)
    for s in range(world):
        pos = np.concatenate([[0], np.cumsum(recv_len[s].numpy())])
        for j in range(n):
            if recv_len[s][j] > 0:
                rr = recv_row[s].numpy()[pos[j]:pos[j + 1]]
                new[rr, j] = recv_val[s].numpy()[pos[j]:pos[j + 1]]
    ok = np.array_equal(new, dense[:, dest[rank]:dest[rank + 1]]) and int(total.sum()) == int(
        np.count_nonzero(dense[:, dest[rank]:dest[rank + 1]]))
    flags = [None] * world
    dist.all_gather_object(flags, (ok, dest))
    if rank == 0:
        out.put(flags)
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_gloo_ranks_all_to_all_reblock():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_a2a_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    flags = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    assert all(ok for ok, _ in flags), flags
    assert flags[0][1] == flags[1][1]  # the same split on both ranks
