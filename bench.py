#!/usr/bin/env python
"""bench.py — pMMF factorization throughput on BASELINE.json config 4.

Workload (BASELINE.json configs[3]): R-MAT scale 20
(n = 1,048,576, 16·n edge samples, a,b,c,d = .57,.19,.19,.05, seed 42),
normalized Laplacian + 1e-2·I (nnz ≈ 3.2e7, fp64), factorized with k=2, P=15,
m=512, eta=0.5, c_min=10, c_max=10000, D_max=500, bypass on, seed 42.
A step = one complete pmmf::factorize (every stage: clustering, reblock,
Gram, search, apply, residual, core) of that matrix.

  value : rotations/s with the input triplets already resident in HBM
          (C-ABI call with device pointers), max step time over ranks.
  e2e   : the same through the C-ABI with HOST buffers: H2D of the triplets
          and D2H of the whole MmfFactorization inside the timed region.
  roofline : the dominant kernel (rotation stream write pass), algorithmic
          bytes per SURVEY.md §8(d) ÷ its CUDA-event time, against the
          measured HBM copy bandwidth (MEASURED_PEAKS.json).
  cpu_baseline : the reference compiled in place (oracle/_ref) on the host
          cores, on a bounded sample of the same recipe (R-MAT scale 14, m=512).

Multi-GPU (--gpus N under torchrun): ONE factorization per step with the
clusters of every stage sharded over the N ranks (shard.cuh: redundant
clustering/reblock, owned clusters' Gram + search + rotation passes, NCCL
exchanges of the rotation slots and column slabs) — strong scaling, the
step time is the max over ranks.  --impl reference runs the reference's CPU
path instead.
"""
import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "pMMF factorization throughput, R-MAT n=1M (config 4)"
UNIT = "rotations/s"

# --workload: config 4 is the headline; the other BASELINE configs print the
# same line shape (their own parity-test cases, timed on request).
WORKLOADS = {
    "c1": {"metric": "pMMF factorization throughput, dense SPD n=1024 (config 1)",
           "desc": "config 1: dense SPD n=1024, X X^T/256 + 1e-3 I", "cpu": "c1"},
    "c3": {"metric": "pMMF factorization throughput, RBF kernel n=16384 k=3 (config 3)",
           "desc": "config 3: RBF kernel n=16384 in 10-D, bandwidth 0.5, + 1e-4 I", "cpu": "c3s"},
    "c4": {"metric": METRIC, "desc": "config 4: R-MAT scale 20 epv 32, normalized Laplacian + 1e-2 I", "cpu": "c4s"},
    "c5": {"metric": "pMMF factorization throughput, anisotropic Poisson 1024^2 (config 5)",
           "desc": "config 5: 5-point anisotropic Poisson 1024x1024 (a_x=100, a_y=1)", "cpu": "c5s"},
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--scale", type=int, default=20, help="R-MAT scale (20 = BASELINE config 4)")
    ap.add_argument("--cpu-scale", type=int, default=14, help="R-MAT scale of the bounded CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--gram", default="seq", choices=["seq", "dmma"],
                    help="dense Gram kernel: bitwise sequential SYRK (default) or FP64 tensor cores (DMMA)")
    ap.add_argument("--launch-list", action="store_true",
                    help="run exactly one factorization step and exit (for the ncu launch list / traffic passes)")
    return ap.parse_args()


def merge_traffic():
    """DRAM bytes (read + write) per launch of the write pass, from the ncu
    dram__bytes pass over every such launch of one factorization
    (profiles/merge_traffic_r01e.json, scripts/gpu_evidence_r01e.sh)."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "merge_traffic_r03.json")
    if not os.path.exists(path):
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "merge_traffic_r02.json")
    if not os.path.exists(path):
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "merge_traffic_r01e.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def reference_full_size(wl):
    """The reference's own full-size run of this config, RECORDED (not timed
    here: 753 s and 183 GB of host RAM on config 4): GPU vs compiled reference
    on the GPU box's 16 host cores, bitwise identical
    (scripts/gpu_parity_fullsize_r03.sh -> profiles/parity_fullsize_r03.jsonl)."""
    want = {"c4": "rmat:20", "c5": "grid:1024"}.get(wl)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "parity_fullsize_r03.jsonl")
    if want is None or not os.path.exists(path):
        return None
    try:
        for ln in open(path):
            d = json.loads(ln)
            if d.get("workload") == want:
                return {"recorded": True, "source": "profiles/parity_fullsize_r03.jsonl", "workload": want,
                        "n": d["n"], "nnz": d["nnz"], "threads": d["threads"], "reference_s": d["ref_s"],
                        "reference_value": d["ref_rot_per_s"], "unit": UNIT, "peak_rss_gb": d["peak_rss_gb"],
                        "gpu_e2e_s_cold_first_call": d["gpu_s"], "bitwise_identical": d["bitwise_identical"]}
    except (OSError, ValueError, KeyError):
        return None
    return None


def config_params(wl="c4"):
    from paper_1507_04396_b200.abi import make_params

    if wl == "c1":
        return make_params(k=2, n_stages=8, eta=0.5, m_target=2, c_min=10, c_max=5000, d_max=500, seed=42)
    if wl in ("c3", "c3s"):
        return make_params(k=3, n_stages=10, eta=0.5, m_target=16, c_min=10, c_max=10000, d_max=500, seed=42)
    if wl in ("c5", "c5s"):
        return make_params(k=2, n_stages=15, eta=0.5, m_target=256, seed=42)
    return make_params(k=2, n_stages=15, eta=0.5, m_target=512, c_min=10, c_max=10000, d_max=500,
                       bypass_enabled=True, core_min=10, core_cap=4096, seed=42)


def workload(scale, wl="c4"):
    from paper_1507_04396_b200 import api

    if wl == "c1":
        return api.workload_dense_spd(1024, 256, 42)
    if wl == "c3":
        return api.workload_rbf(16384, seed=42)
    if wl == "c3s":  # the CPU reference's feasible size
        return api.workload_rbf(2048, seed=42)
    if wl == "c5":
        return api.workload_aniso_grid(1024)
    if wl == "c5s":
        return api.workload_aniso_grid(256)
    return api.workload_rmat(scale, 32, 42, 1e-2)


def cpu_sample_desc(wl, scale):
    return {"c1": "dense SPD n=1024 (full config 1)",
            "c3s": "RBF n=2048 (config-3 recipe; n=16384 needs ~275 GB per Gram buffer on the CPU path)",
            "c5s": "anisotropic Poisson 256x256, m=256 (config-5 recipe at 1/16 of the grid)",
            "c4s": f"R-MAT scale {scale}, epv 32, m=512 (config-4 recipe at n=2^{scale}); the reference cannot "
                   f"hold n=2^20 (OOM, SURVEY.md §6)"}[wl]


def fp64_peak():
    """cuBLAS DGEMM (torch.matmul fp64, 8192^3, best of 5) on this GPU, TFLOP/s."""
    import torch

    a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    torch.matmul(a, b)
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2 * 8192 ** 3 / (best / 1e3) / 1e12


class Clocks:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        if os.environ.get("BENCH_NO_CLOCKS"):  # experiments only: no sampler process
            self.proc = None
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms",
                 os.environ.get("BENCH_CLOCK_MS", "200")],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.first = threading.Event()
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's start-up (NVML init) costs host CPU for ~0.1-0.2 s:
            # let it finish before the timed region (launch-bound configs
            # otherwise lose their first timed step to it)
            self.first.wait(timeout=10)
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))
            self.first.set()
        self.first.set()

    def mark(self, begin=True):
        """Bounds of the timed region: only samples inside it are reported
        (the sampler starts before the warm-up, so its start-up cost never
        lands in a timed step)."""
        if begin:
            self.t0 = time.perf_counter()
        else:
            self.t1 = time.perf_counter()

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = getattr(self, "t0", None), getattr(self, "t1", None)
        inside = [ln for t, ln in self.lines if (t0 is None or t >= t0) and (t1 is None or t <= t1 + 0.25)]
        for ln in inside or [ln for _, ln in self.lines[-3:]]:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ref_workload(scale, wl="c4"):
    """The same seeded recipes on the reference's own pmmf::Rng (oracle/_ref),
    so the reference arm never loads libpmmf_b200.so (tests/test_workloads.py
    checks both generators emit identical triplets)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracles

    if wl == "c1":
        return oracles.ref_workload("dense_spd", 1024, 256, 42, 1e-3)
    if wl == "c3":
        return oracles.ref_workload("rbf", 16384, 10, 0.5, 42, 1e-4)
    if wl == "c3s":
        return oracles.ref_workload("rbf", 2048, 10, 0.5, 42, 1e-4)
    if wl == "c5":
        return oracles.ref_workload("aniso_grid", 1024, 100.0, 1.0)
    if wl == "c5s":
        return oracles.ref_workload("aniso_grid", 256, 100.0, 1.0)
    return oracles.ref_workload("rmat", scale, 32, 42, 1e-2)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def cpu_reference_run(scale, threads, steps=1, warmup=0, wl="c4", inp=None):
    """The reference compiled in place (oracle/_ref, pmmf::factorize) on a
    bounded sample of the workload; input from the reference's own Rng."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracles

    ref = oracles.load("ref")
    ref.lib.pmmf_ref_set_threads(threads)
    cw = WORKLOADS[wl]["cpu"]
    if inp is None:
        inp = ref_workload(scale, cw)
    params = config_params(cw)
    times, rots = [], 0
    for i in range(warmup + steps):
        t = time.perf_counter()
        f = oracles.factorize("ref", inp, params)
        dt = time.perf_counter() - t
        rots = sum(len(s.rot_indices) for s in f.stages)
        if i >= warmup:
            times.append(dt)
    return rots, times, inp


DATA = "synthetic (seeded SURVEY.md §8(d) recipes, s_in = 42); inputs > L2 (no flush needed)"


def config_dict(args, W, n, nnz, params, world):
    """The workload both arms report (the reference arm times a bounded
    sample of it, described in its cpu_baseline.sample)."""
    return {"dense_gram": getattr(args, "gram", "seq"),"workload": W["desc"] if args.workload != "c4" else
            f"config 4: R-MAT scale {args.scale} epv 32, normalized Laplacian + 1e-2 I",
            "n": int(n), "nnz": int(nnz), "k": int(params.k), "P": int(params.n_stages),
            "m": int(params.m_target), "c_max": int(params.c_max),
            "parallelism": f"clusters sharded x{world}" if world > 1 else "single GPU",
            "l2": "working set >> 126 MB L2"}


def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")
    return world, rank, local, dist


def time_mmf_apply(lib, coo_dev, params, err, n):
    """MmfOperator inv_sqrt apply (the CG preconditioner, transform_ops.hpp:51-67)
    on device-resident vectors: 1 and 20 rhs, CUDA events, best of 10.
    Algorithmic bytes: 2 R_nid (8k^2+4k) + 2*2*8 n b + 8 g^2."""
    import torch
    from paper_1507_04396_b200 import abi

    h = ctypes.c_void_p()
    abi.raise_for(lib.factorize(ctypes.byref(coo_dev), ctypes.byref(params), ctypes.byref(h), err, len(err)), err)
    f = lib.read_result(h)
    op = ctypes.c_void_p()
    abi.raise_for(lib.operator_create(h, 1e-12, ctypes.byref(op), err, len(err)), err)
    lib.result_free(h)
    k = int(params.k)
    ident = np.eye(k).reshape(-1)
    r_nid = 0
    for st in f.stages:
        q = st.rot_matrices.reshape(len(st.rot_matrices), -1)
        r_nid += int(np.sum(~np.all(q == ident, axis=1)))
    g = len(f.core_indices)
    out = {"rotations_non_identity": r_nid, "core": g}
    peak, _ = peaks()
    for b in (1, 20):
        v = torch.randn(b, n, dtype=torch.float64, device="cuda")
        o = torch.empty_like(v)
        best = 1e30
        for i in range(12):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            abi.raise_for(lib.operator_apply(op, 2, b, v.data_ptr(), o.data_ptr(), 1, err, len(err)), err)
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                best = min(best, e0.elapsed_time(e1))
        by = 2 * r_nid * (8 * k * k + 4 * k) + 2 * 2 * 8 * n * b + 8 * g * g
        out[f"rhs{b}"] = {"ms": best, "algorithmic_bytes": by, "achieved_GBs": by / 1e9 / (best / 1e3),
                          "frac_hbm": by / 1e9 / (best / 1e3) / peak,
                          "note": "includes the rhs-major <-> index-major transposes of the public call"}
    lib.operator_free(op)
    return out


def cg_block(lib, coo_dev, params, err, cpu_threads):
    """Config 5's CG (run_solve_experiment + pmmf_preconditioner, solver.hpp:
    343-416; SURVEY.md §8(d) "CG time per iteration on the same RHS set"):
      * GPU at full size: 20 seeded rhs, tol 1e-8, a bounded 400 iterations
        (convergence takes ~5,500; per-iteration time is the metric);
      * the reference (oracle/_ref, all host threads, rhs in parallel as its
        run_solve_experiment does) and the GPU on the 256^2 sample to
        convergence: same input, same rhs set.
    per_iteration_ms = wall / sum of iterations over the rhs (the reference's
    SolveReport::per_iteration_ms), plus the batched GPU figure
    wall / max iterations (all 20 rhs advance together)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracles
    from paper_1507_04396_b200 import abi

    def run(which, handle_lib, coo, op, nr, max_iter):
        cfg = abi.SolveConfig(1e-8, max_iter, nr, 0)
        it = np.zeros(nr, np.int32)
        cv = np.zeros(nr, np.int32)
        bk = np.zeros(nr, np.int32)
        tr = np.zeros((nr, max_iter + 1))
        wall = ctypes.c_double()
        e = handle_lib.errbuf()
        abi.raise_for(handle_lib.solve(ctypes.byref(coo), op, ctypes.byref(cfg), it.ctypes.data_as(abi.c_i32p),
                                       cv.ctypes.data_as(abi.c_i32p), bk.ctypes.data_as(abi.c_i32p),
                                       tr.ctypes.data_as(abi.c_f64p), ctypes.byref(wall), e, len(e)), e)
        tot = int(it.sum())
        return {"impl": which, "rhs": nr, "iterations_mean": float(it.mean()), "iterations_max": int(it.max()),
                "converged": int(cv.sum()), "wall_ms": wall.value,
                "per_iteration_ms": wall.value / tot if tot else None,
                "batched_iteration_ms": wall.value / int(it.max()) if it.max() else None,
                "final_rel_residual_mean": float(np.mean([tr[r, it[r]] / tr[r, 0] for r in range(nr)]))}

    out = {}
    h = ctypes.c_void_p()
    abi.raise_for(lib.factorize(ctypes.byref(coo_dev), ctypes.byref(params), ctypes.byref(h), err, len(err)), err)
    op = ctypes.c_void_p()
    abi.raise_for(lib.operator_create(h, 1e-12, ctypes.byref(op), err, len(err)), err)
    lib.result_free(h)
    # full size: the triplets on the device (the solve builds its CSR there)
    out["gpu_full_1024x1024"] = run("gpu", lib, coo_dev, op, 20, 400)
    short = run("gpu", lib, coo_dev, op, 20, 100)
    # the marginal iteration (setup excluded: CSR build, 20 x n host rhs draws)
    out["gpu_full_1024x1024"]["marginal_iteration_ms"] = (out["gpu_full_1024x1024"]["wall_ms"] - short["wall_ms"]) / 300
    out["gpu_full_1024x1024"]["note"] = ("bounded at 400 iterations (full convergence ~5,500); marginal_iteration_ms = "
                                         "(wall(400) - wall(100)) / 300, all 20 rhs advancing together")
    lib.operator_free(op)
    # 256^2 sample, both arms, to convergence
    inp = ref_workload(0, "c5s")
    p = config_params("c5s")
    for which in ("ref", "gpu"):
        L = oracles.load(which)
        if which == "ref":
            L.lib.pmmf_ref_set_threads(cpu_threads)
        _, hh = oracles.result_handle(which, inp, p)
        o = ctypes.c_void_p()
        e = L.errbuf()
        abi.raise_for(L.operator_create(hh, 1e-12, ctypes.byref(o), e, len(e)), e)
        L.result_free(hh)
        coo, keep = abi.make_coo(*inp)
        r = run(which, L, coo, o, 20, 5000)
        L.operator_free(o)
        out[f"{which}_256x256"] = r
    out["cores"] = cpu_threads
    out["cpu_model"] = cpu_model()
    return out


def like_for_like(lib, inp, cw, cpu_rots, cpu_s, err, steps=5):
    """The GPU on the reference's exact sample input (same triplets, same
    params): e2e through the C-ABI with host buffers (H2D of the triplets and
    D2H of the whole factorization inside the step, as the reference returns
    a host MmfFactorization), best of `steps` after 2 warm-ups (the reference's
    time is its best run too)."""
    import torch
    from paper_1507_04396_b200 import abi

    params = config_params(cw)
    n, rows, cols, vals = inp
    pinned = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in (rows, cols, vals)]
    coo, keep = abi.make_coo(n, *(t.numpy() for t in pinned))
    ts, rots = [], 0
    for i in range(2 + steps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        h = ctypes.c_void_p()
        abi.raise_for(lib.factorize(ctypes.byref(coo), ctypes.byref(params), ctypes.byref(h), err, len(err)), err)
        f = lib.read_result(h)
        lib.result_free(h)
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(time.perf_counter() - t)
        rots = sum(len(st.rot_indices) for st in f.stages)
    # the same statistic on both sides: the reference's time is its best run
    # (cpu_baseline), so the GPU's is the best of its steps; the mean rides along
    g = min(ts)
    return {"input": f"the cpu_baseline sample (n={n}, nnz={len(vals)})", "rotations": rots,
            "same_rotation_count": rots == cpu_rots, "statistic": f"best of {len(ts)} (GPU) / best run (reference)",
            "gpu_e2e_s": g, "gpu_e2e_mean_s": sum(ts) / len(ts), "gpu_value": rots / g, "reference_s": cpu_s,
            "reference_value": cpu_rots / cpu_s, "speedup": cpu_s / g, "unit": UNIT}


def main():
    args = parse()
    W = WORKLOADS[args.workload]
    world, rank, local, dist = dist_init(args)
    if args.impl == "reference":
        if rank != 0:
            return
        threads = os.cpu_count() or 1
        full = ref_workload(args.scale, args.workload)  # for the config only (n, nnz)
        params = config_params(args.workload)
        cfg = config_dict(args, W, full[0], len(full[3]), params, world)
        del full
        rots, times, inp = cpu_reference_run(args.cpu_scale, threads, steps=args.steps, warmup=args.warmup,
                                             wl=args.workload)
        mean = sum(times) / len(times)  # the same statistic as the GPU arm (total over K steps / K)
        v = rots / mean
        sample = cpu_sample_desc(W["cpu"], args.cpu_scale) + f" (n={inp[0]}, nnz={len(inp[1])}, {rots} rotations)"
        line = {"metric": W["metric"], "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": mean * 1e3, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": DATA, "impl": "reference",
                "config": cfg,
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                                 "cpu_model": cpu_model(),
                                 "sample": "each step: pmmf::factorize (oracle/_ref, -O2, all host threads) on "
                                           + sample + "; input from the reference's own pmmf::Rng",
                                 "step_s": [round(t, 3) for t in times],
                                 "min_s": min(times), "median_s": float(np.median(times))},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch

    torch.cuda.set_device(local)
    from paper_1507_04396_b200 import abi, api

    lib = api.library()
    L = lib.lib
    L.pmmf_b200_profile_read.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_double)]
    L.pmmf_b200_profile_enable.argtypes = [ctypes.c_int32]
    params = config_params(args.workload)
    api.set_dense_gram(1 if args.gram == "dmma" else 0)
    n, rows, cols, vals = workload(args.scale, args.workload)
    d_rows = torch.from_numpy(rows).cuda()
    d_cols = torch.from_numpy(cols).cuda()
    d_vals = torch.from_numpy(vals).cuda()
    torch.cuda.synchronize()
    coo_dev, keep_dev = abi.make_coo(n, d_rows, d_cols, d_vals, on_device=True, device=local)
    # e2e input: host buffers in pinned memory (the contract's "copy of that
    # step's inputs from pinned host memory"), copied by the library each step
    pinned = [torch.from_numpy(x).pin_memory() for x in (rows, cols, vals)]
    coo_host, keep_host = abi.make_coo(n, *(t.numpy() for t in pinned), device=local)
    err = lib.errbuf()
    # N > 1: the clusters of every stage sharded over the ranks (NCCL)
    comm = api.Communicator.from_torch_distributed(local) if world > 1 else None

    def factorize(coo, h):
        if comm is None:
            return lib.factorize(ctypes.byref(coo), ctypes.byref(params), ctypes.byref(h), err, len(err))
        return L.pmmf_b200_factorize_sharded(ctypes.byref(coo), ctypes.byref(params), comm.handle, ctypes.byref(h),
                                             err, len(err))

    last_phases = np.zeros(6)

    def run_device():
        h = ctypes.c_void_p()
        abi.raise_for(factorize(coo_dev, h), err)
        s = abi.Summary()
        lib.result_summary(h, ctypes.byref(s))
        ph = np.zeros(6)
        info = np.zeros((max(s.n_stages, 1), 7), np.int64)
        lib.result_stats(h, ph.ctypes.data_as(abi.c_f64p), info.ctypes.data_as(abi.c_i64p))
        last_phases[:] = ph
        rots = 0
        for st in range(s.n_stages):
            sz = abi.StageSizes()
            lib.result_stage_sizes(h, st, ctypes.byref(sz))
            rots += sz.n_rotations
        lib.result_free(h)
        return rots

    def run_e2e():
        h = ctypes.c_void_p()
        abi.raise_for(factorize(coo_host, h), err)
        f = lib.read_result(h)
        lib.result_free(h)
        out_bytes = sum(a.nbytes for st in f.stages for a in (st.cluster_offsets, st.members, st.rot_indices, st.rot_matrices,
                                                              st.elim_index, st.elim_diagonal, st.elim_off_mass_sq, st.bypassed))
        out_bytes += f.core.nbytes + f.core_indices.nbytes + f.diag_index.nbytes + f.diag_value.nbytes
        return sum(len(st.rot_indices) for st in f.stages), out_bytes

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    if args.launch_list:
        run_device()
        torch.cuda.synchronize()
        return
    L.pmmf_b200_profile_enable(0)
    clocks = Clocks(local)
    clocks.start()  # nvidia-smi's start-up overlaps the warm-up
    for _ in range(args.warmup):
        run_device()
    # ---- timed region: device-resident input, live kernel accounting OFF
    # (its per-level events would count toward the step); the roofline
    # counters come from one extra profiled step after the timed region.
    barrier()
    torch.cuda.synchronize()
    clocks.mark(True)
    launches0 = api.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step_ms, rots = [], 0
    step_phases = []
    for _ in range(args.steps):
        ev0.record()
        rots = run_device()
        ev1.record()
        torch.cuda.synchronize()
        step_ms.append(ev0.elapsed_time(ev1))
        step_phases.append([round(float(x), 1) for x in last_phases])
    launches = api.kernel_launches() - launches0
    barrier()
    torch.cuda.synchronize()
    clocks.mark(False)
    clk = clocks.stop()
    timed_phases = last_phases.copy()
    # roofline pass: one untimed step with the per-launch CUDA events on
    L.pmmf_b200_profile_enable(1)
    prof_step_ms = time.perf_counter()
    run_device()
    torch.cuda.synchronize()
    prof_step_ms = (time.perf_counter() - prof_step_ms) * 1e3
    prof = {}
    for name in ("rotate_write", "rotate_count", "gram_dense", "gram_dmma"):
        c, ms, by = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
        if L.pmmf_b200_profile_read(name.encode(), ctypes.byref(c), ctypes.byref(ms), ctypes.byref(by)) == 0:
            prof[name] = (c.value, ms.value, by.value)
    L.pmmf_b200_profile_enable(0)
    total_ms = max_over_ranks(sum(step_ms))
    ms_per_step = total_ms / args.steps
    value = rots / (ms_per_step / 1e3)  # one factorization per step for the whole job

    # ---- e2e: host buffers through the C-ABI, H2D + D2H inside the step
    barrier()
    e2e_ms = []
    out_bytes = 0
    for _ in range(max(1, min(args.steps, 10))):
        torch.cuda.synchronize()
        t = time.perf_counter()
        _, out_bytes = run_e2e()
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t) * 1e3)
    e2e_step = max_over_ranks(sum(e2e_ms) / len(e2e_ms))
    e2e = {"value": rots / (e2e_step / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": int(rows.nbytes + cols.nbytes + vals.nbytes), "d2h_bytes_per_step": int(out_bytes),
           "ms_per_step": e2e_step}

    peak, peak_src = peaks()
    roof = None
    if "rotate_write" in prof:
        c, ms, by = prof["rotate_write"]
        achieved = (by / 1e9) / (ms / 1e3) if ms > 0 else 0.0
        roof = {"bound": "hbm", "kernel": "k_merge2<true> (k = 2 rotation stream, write pass)", "achieved": achieved,
                "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": merge_traffic() if args.workload == "c4" else None,
                "launches": c, "kernel_ms_total": ms, "algorithmic_bytes_total": by, "peak_source": peak_src,
                "share_of_step": ms / prof_step_ms,
                "measured_in": "one extra profiled step after the timed region (CUDA events per launch)"}
        if "rotate_count" in prof:
            c2, ms2, by2 = prof["rotate_count"]
            roof["count_pass"] = {"launches": c2, "ms": ms2, "achieved_GBs": (by2 / 1e9) / (ms2 / 1e3) if ms2 else 0.0}

    gname = "gram_dmma" if args.gram == "dmma" else "gram_dense"
    if args.workload == "c3" and gname in prof:
        # dense Gram against cuBLAS DGEMM: the bitwise sequential SYRK on the
        # FP64 pipe, or the DMMA tensor-core SYRK (--gram dmma)
        c, ms, fl = prof[gname]
        tf = (fl / 1e12) / (ms / 1e3) if ms > 0 else 0.0
        pk = fp64_peak()
        kname = ("k_syrk_dmma (dense Gram, FP64 tensor cores: DMMA m8n8k4, TMA-staged)" if args.gram == "dmma" else
                 "k_syrk_seq (dense Gram, sequential row order, unfused mul/add)")
        roof = {"bound": "tensor" if args.gram == "dmma" else "fp64", "kernel": kname,
                "achieved": tf, "peak": pk, "unit": "TFLOP/s", "frac": tf / pk, "traffic": None, "launches": c,
                "kernel_ms_total": ms, "algorithmic_flops_total": fl,
                "peak_source": "measured live: cuBLAS DGEMM (torch.matmul fp64 8192^3, best of 5)",
                "share_of_step": ms / prof_step_ms, "write_pass": roof}

    apply = None
    cg = None
    if args.workload == "c5":
        apply = time_mmf_apply(lib, coo_dev, params, err, n)
        if rank == 0 and not args.no_cpu_baseline:
            try:
                cg = cg_block(lib, coo_dev, params, err, os.cpu_count() or 1)
            except Exception as e:  # the checker is optional on the box
                import traceback
                cg = {"unavailable": f"{e!r}: {traceback.format_exc()[-600:]}"}

    cpu, like = None, None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            # best of 3 when the sample is short (SURVEY.md §8(d) "Repeats")
            crots, ctimes, cinp = cpu_reference_run(args.cpu_scale, threads, steps=1, wl=args.workload)
            if ctimes[0] < 20.0:
                crots, more, _ = cpu_reference_run(args.cpu_scale, threads, steps=2, wl=args.workload, inp=cinp)
                ctimes += more
            cbest = min(ctimes)
            cpu = {"value": crots / cbest, "unit": UNIT, "cores": threads, "kind": "reference",
                   "cpu_model": cpu_model(),
                   "sample": f"reference (oracle/_ref, pmmf::factorize, -O2 -ffp-contract=off) on "
                             f"{cpu_sample_desc(W['cpu'], args.cpu_scale)} (n={cinp[0]}, nnz={len(cinp[1])}, "
                             f"{crots} rotations), best of {len(ctimes)}: {cbest:.2f} s, {threads} threads",
                   "runs_s": [round(t, 3) for t in ctimes]}
            like = like_for_like(lib, cinp, W["cpu"], crots, cbest, err)
        except Exception as e:  # the checker is optional on the box
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {"metric": W["metric"], "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": DATA,
                "config": config_dict(args, W, n, len(vals), params, world), "rotations_per_step": int(rots),
                "roofline": roof, "cpu_baseline": cpu, "like_for_like": like,
                "reference_full_size": reference_full_size(args.workload), "e2e": e2e, "gpu_launches": int(launches),
                "mmf_apply": apply, "cg": cg,
                "clocks": clk, "step_ms": step_ms,
                "phases_ms_steps": step_phases,  # [clustering, gram, search, apply, reblock, total] per timed step
                "phases_ms_last_step": dict(zip(["clustering", "gram", "search", "apply", "reblock", "total"],
                                                [round(float(x), 1) for x in timed_phases]))}
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
