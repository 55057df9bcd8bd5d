"""Modelled multi-GPU step time of the sharded factorization from ONE GPU.

Only one B200 is reachable this round, so the N-GPU step is assembled from
measured parts: a config-N factorization with W virtual ranks
(api.Communicator(W, virtual=True)) runs every rank's sharded work one after
another on this GPU, and PMMF_B200_SHARD_TIMING reports each rank's Gram+search and
slab apply time per stage.  Then

  T_W = T_virtual - sum_s sum_r (gs_rs + ap_rs) + sum_s (max_r gs_rs + max_r ap_rs) + X_W

(the sharded clustering scorer's calls enter the same way: sum over ranks
out, max over ranks in)

where the clustering/reblock/bookkeeping remainder is replicated on every
rank and X_W is the slab exchange: every rank receives the other ranks'
slabs, 12 B x nnz(A'') x (W-1)/W per stage, at an assumed NCCL broadcast
ingress of B GB/s per GPU (--nvlink-gbs, default 400 of NVLink 5's 900).
The result is also checked bit-for-bit against the one-GPU factorization.

usage: python scripts/shard_model.py [--workload c4] [--worlds 2 4 8]
Prints one JSON object (profiles/shard_model_r01.json is this output).
"""
import argparse
import json
import os
import re
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def child(wl, world, out):
    """One factorization (world 0 = plain single-GPU entry point)."""
    import ctypes

    import numpy as np

    import bench
    from paper_1507_04396_b200 import abi, api

    lib = api.library()
    params = bench.config_params(wl)
    n, rows, cols, vals = bench.workload(20, wl)
    coo, keep = abi.make_coo(n, rows, cols, vals)
    comm = api.Communicator(world, virtual=True) if world > 0 else None
    err = lib.errbuf()
    res = {}
    for it in range(2):  # first run maps the memory pool; time the second
        h = ctypes.c_void_p()
        t = time.perf_counter()
        st = (lib.factorize(ctypes.byref(coo), ctypes.byref(params), ctypes.byref(h), err, len(err)) if comm is None
              else lib.lib.pmmf_b200_factorize_sharded(ctypes.byref(coo), ctypes.byref(params), comm.handle,
                                                       ctypes.byref(h), err, len(err)))
        abi.raise_for(st, err)
        wall = (time.perf_counter() - t) * 1e3
        f = lib.read_result(h)
        lib.result_free(h)
        res = {"wall_ms": wall, "rotations": int(sum(len(s.rot_indices) for s in f.stages)),
               "digest": digest(f)}
        sys.stderr.flush()
        os.write(2, b"[model] run-end\n")
    with open(out, "w") as fh:
        json.dump(res, fh)


def digest(f):
    import hashlib

    import numpy as np

    h = hashlib.sha256()
    for st in f.stages:
        for a in (st.cluster_offsets, st.members, st.rot_indices, st.rot_matrices, st.elim_index, st.elim_diagonal,
                  st.elim_off_mass_sq):
            h.update(np.ascontiguousarray(a).tobytes())
    h.update(np.ascontiguousarray(f.core).tobytes())
    h.update(np.float64(f.residual_sq).tobytes())
    return h.hexdigest()


def run(wl, world, trace):
    out = f"/tmp/shard_model_{wl}_{world}.json"
    env = dict(os.environ)
    if trace:
        env["PMMF_B200_SHARD_TIMING"] = "1"
    p = subprocess.run([sys.executable, __file__, "--child", wl, str(world), out], env=env, capture_output=True,
                       text=True, cwd=ROOT)
    if p.returncode != 0:
        raise RuntimeError(p.stderr[-3000:])
    with open(out) as fh:
        res = json.load(fh)
    # keep only the timed (second) run's trace
    log = p.stderr.split("[model] run-end\n")
    res["trace"] = log[1] if len(log) > 2 else p.stderr
    return res


def model(res, world, gbs):
    """Owned-column design (shard.cuh): per stage, the max over ranks of
    every sharded part (scoring calls, slab reblock, Gram+search, slab
    apply) replaces their sum; the in-process slab exchange of the virtual
    run is replaced by the all-to-all at `gbs` GB/s of per-rank ingress."""
    tr = res["trace"]
    gs, ap, rb = {}, {}, {}
    for m in re.finditer(r"shard stage (\d+) rank (\d+): gram\+search ([\d.]+) ms \(([\d.]+) wall\)", tr):
        gs[(int(m[1]), int(m[2]))] = float(m[4])
    for m in re.finditer(r"shard stage (\d+) rank (\d+): apply ([\d.]+) ms, slab (\d+) entries", tr):
        ap[(int(m[1]), int(m[2]))] = float(m[3])
    for m in re.finditer(r"shard stage (\d+) rank (\d+): reblock ([\d.]+) ms", tr):
        rb[(int(m[1]), int(m[2]))] = float(m[3])
    xv = sum(float(m[1]) for m in re.finditer(r"shard stage \d+: exchange ([\d.]+) ms", tr))
    ingress = [int(m[1]) for m in re.finditer(r"shard stage \d+: all-to-all ingress max (\d+) bytes", tr)]
    serial = sum(gs.values()) + sum(ap.values()) + sum(rb.values()) + xv
    par = 0.0
    sc_sum = sc_max = 0.0
    for m in re.finditer(r"shard score: (\d+) ranks, sum ([\d.]+) ms, max ([\d.]+) ms", tr):
        sc_sum += float(m[2])
        sc_max += float(m[3])
    serial += sc_sum
    par += sc_max
    stages = sorted({s for s, _ in gs} | {s for s, _ in ap} | {s for s, _ in rb})
    per_stage = []
    for s in stages:
        g = [gs.get((s, r), 0.0) for r in range(world)]
        a = [ap.get((s, r), 0.0) for r in range(world)]
        b = [rb.get((s, r), 0.0) for r in range(world)]
        par += max(g) + max(a) + max(b)
        per_stage.append({"stage": s, "gram_search_ms": [round(x, 2) for x in g], "apply_ms": [round(x, 2) for x in a],
                          "reblock_ms": [round(x, 2) for x in b]})
    xms = sum(ingress) / (gbs * 1e9) * 1e3
    t = res["wall_ms"] - serial + par + xms
    return {"virtual_wall_ms": res["wall_ms"], "sharded_serial_ms": serial, "sharded_max_over_ranks_ms": par,
            "scoring_sum_ms": sc_sum, "scoring_max_ms": sc_max, "virtual_exchange_ms": xv,
            "replicated_ms": res["wall_ms"] - serial, "all_to_all_bytes_max_rank": sum(ingress),
            "exchange_ms_modelled": xms, "modelled_step_ms": t, "per_stage": per_stage}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--worlds", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--nvlink-gbs", type=float, default=400.0)
    ap.add_argument("--child", nargs=3)
    a = ap.parse_args()
    if a.child:
        child(a.child[0], int(a.child[1]), a.child[2])
        return
    base = run(a.workload, 0, trace=False)
    out = {"workload": a.workload, "rotations": base["rotations"], "one_gpu_wall_ms": base["wall_ms"],
           "one_gpu_rotations_per_s": base["rotations"] / base["wall_ms"] * 1e3, "nvlink_gbs_assumed": a.nvlink_gbs,
           "note": "owned-column slabs: modelled from single-GPU virtual-rank runs (one sync per rank and "
                   "phase); all-to-all reblock time = max per-rank ingress bytes / assumed NCCL bandwidth",
           "worlds": {}}
    for w in a.worlds:
        res = run(a.workload, w, trace=True)
        m = model(res, w, a.nvlink_gbs)
        m["bit_identical_to_one_gpu"] = res["digest"] == base["digest"]
        m["modelled_rotations_per_s"] = base["rotations"] / m["modelled_step_ms"] * 1e3
        m["modelled_speedup"] = base["wall_ms"] / m["modelled_step_ms"]
        out["worlds"][str(w)] = m
    print(json.dumps(out))


if __name__ == "__main__":
    main()
