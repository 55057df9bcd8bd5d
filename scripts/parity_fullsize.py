#!/usr/bin/env python
"""Parity of the GPU factorization against the reference compiled in place
(oracle/_ref, pmmf::factorize) at config-4 sizes the CPU reference can only
run on a host with a lot of RAM (the GPU box: 196 GB, 16 cores).

  python scripts/parity_fullsize.py gpu WL OUT.npz   # GPU factorization -> npz
  python scripts/parity_fullsize.py ref WL OUT.npz   # reference, compare with OUT.npz

WL is rmat:SCALE (config 4's recipe, m=512) or grid:SIDE (config 5's, m=256).

The two halves run in separate processes so the reference's process can run
under a memory limit (ulimit -v) without CUDA in it.  Input: config 4's recipe
(R-MAT epv 32, seed 42, m=512, c_max=10^4) at R-MAT scale SCALE, generated on
the reference's own pmmf::Rng for the reference half and on the library's
generator for the GPU half (identical triplets, tests/test_workloads.py).
Prints one JSON line with wall times, rotation counts, peak RSS and the
bitwise verdict field by field.
"""
import json
import os
import resource
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

FIELDS = ["cluster_offsets", "members", "rot_indices", "rot_matrices", "elim_index", "elim_diagonal",
          "elim_off_mass_sq", "bypassed"]


def params(wl):
    from paper_1507_04396_b200.abi import make_params

    if wl.startswith("grid"):
        return make_params(k=2, n_stages=15, eta=0.5, m_target=256, seed=42)
    return make_params(k=2, n_stages=15, eta=0.5, m_target=512, c_min=10, c_max=10000, d_max=500,
                       bypass_enabled=True, core_min=10, core_cap=4096, seed=42)


def flat_to_npz(f, path, extra):
    d = {"n": f.n, "residual_sq": f.residual_sq, "core": f.core, "core_indices": f.core_indices,
         "diag_index": f.diag_index, "diag_value": f.diag_value, "active_history": f.active_history,
         "n_stages": len(f.stages)}
    for s, st in enumerate(f.stages):
        for k in FIELDS:
            d[f"s{s}_{k}"] = getattr(st, k)
    np.savez(path, **d)
    with open(path + ".json", "w") as fh:
        json.dump(extra, fh)


def main():
    which, wl, out = sys.argv[1], sys.argv[2], sys.argv[3]
    size = int(wl.split(":")[1])
    import oracles

    if which == "gpu":
        from paper_1507_04396_b200 import api

        inp = api.workload_aniso_grid(size) if wl.startswith("grid") else api.workload_rmat(size, 32, 42, 1e-2)
        oracles.factorize("gpu", inp, params(wl))  # warm
        t = time.perf_counter()
        f = oracles.factorize("gpu", inp, params(wl))
        dt = time.perf_counter() - t
        rots = sum(len(s.rot_indices) for s in f.stages)
        flat_to_npz(f, out, {"gpu_s": dt, "rotations": rots, "nnz": len(inp[3])})
        print(json.dumps({"which": "gpu", "workload": wl, "n": inp[0], "nnz": len(inp[3]), "gpu_s": dt,
                          "rotations": rots}), flush=True)
        return
    threads = os.cpu_count() or 1
    oracles.load("ref").lib.pmmf_ref_set_threads(threads)
    t0 = time.perf_counter()
    inp = (oracles.ref_workload("aniso_grid", size, 100.0, 1.0) if wl.startswith("grid")
           else oracles.ref_workload("rmat", size, 32, 42, 1e-2))
    gen_s = time.perf_counter() - t0
    t = time.perf_counter()
    f = oracles.factorize("ref", inp, params(wl))
    ref_s = time.perf_counter() - t
    rss_gb = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6
    g = np.load(out)
    meta = json.load(open(out + ".json"))
    diffs = []
    if int(g["n_stages"]) != len(f.stages):
        diffs.append("n_stages")
    for s, st in enumerate(f.stages[: int(g["n_stages"])]):
        for k in FIELDS:
            a, b = g[f"s{s}_{k}"], getattr(st, k)
            if not (a.shape == b.shape and np.array_equal(a, b)):
                diffs.append(f"stage {s + 1} {k}")
    for k in ["core", "core_indices", "diag_index", "diag_value", "active_history"]:
        if not np.array_equal(g[k], getattr(f, k)):
            diffs.append(k)
    if float(g["residual_sq"]) != f.residual_sq:
        diffs.append("residual_sq")
    rots = sum(len(s.rot_indices) for s in f.stages)
    line = {"which": "ref-vs-gpu", "workload": wl, "n": inp[0], "nnz": len(inp[3]), "threads": threads,
            "ref_s": ref_s, "ref_rot_per_s": rots / ref_s, "gen_s": gen_s, "peak_rss_gb": rss_gb,
            "rotations": rots, "gpu_rotations": meta["rotations"], "gpu_s": meta["gpu_s"],
            "gpu_rot_per_s": meta["rotations"] / meta["gpu_s"], "speedup": ref_s / meta["gpu_s"],
            "stages": len(f.stages), "bitwise_identical": not diffs, "diffs": diffs[:20],
            "residual_sq": f.residual_sq, "ref_phases_ms": [float(x) for x in f.phases]}
    print(json.dumps(line), flush=True)
    sys.exit(0 if not diffs else 1)


if __name__ == "__main__":
    main()
