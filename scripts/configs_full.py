"""Full-size runs of BASELINE.json configs 1, 3 and 5 on one GPU (timings only).

  python scripts/configs_full.py c1 c3 c5 [--rhs R] [--max-iter M]

c1: dense SPD n=1024, m=2, P=8.   c3: RBF n=16,384 k=3 P=10 m=16 c_max 1e4.
c5: anisotropic Poisson 1024^2 (a_x=100), m=256, then PCG with the MMF
    inv_sqrt preconditioner on R seeded rhs to 1e-8, plus apply throughput.
"""
import argparse
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1507_04396_b200 import abi, api
from paper_1507_04396_b200.api import BlockedSparseMatrix, ClusterParams, FactorizeParams


def run_factorize(tag, inp, p, reps=2):
    m = BlockedSparseMatrix.from_triplets(*inp)
    for rep in range(reps):
        t = time.time()
        f = api.factorize(m, p)
        wall = time.time() - t
        rots = sum(len(s.rot_indices) for s in f.stages)
        print(f"{tag}: n={inp[0]} nnz={len(inp[1])} wall={wall:.3f}s rotations={rots} rot/s={rots / wall:.0f} "
              f"stages={len(f.stages)} core={len(f.core_indices)} residual_sq={f.residual_sq:.9e}", flush=True)
        print("   phases ms (clustering, gram, search, apply, reblock, total):", np.round(f.phases, 1), flush=True)
    return f


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfgs", nargs="*", default=["c1", "c3", "c5"])
    ap.add_argument("--rhs", type=int, default=20)
    ap.add_argument("--max-iter", type=int, default=20000)
    ap.add_argument("--no-pcg", action="store_true")
    ap.add_argument("--apply-only", action="store_true", help="c5: skip the factorization timing runs")
    args = ap.parse_args()
    for c in args.cfgs:
        if c == "c1":
            run_factorize("c1", api.workload_dense_spd(1024, 256, 42),
                          FactorizeParams(seed=42, n_stages=8, cluster=ClusterParams(m_target=2)))
        elif c == "c3":
            t = time.time()
            inp = api.workload_rbf(16384, seed=42)
            print(f"c3 input generated in {time.time() - t:.1f}s", flush=True)
            run_factorize("c3", inp, FactorizeParams(seed=42, k=3, n_stages=10,
                                                     cluster=ClusterParams(m_target=16, c_max=10000)))
        elif c == "c5":
            inp = api.workload_aniso_grid(1024)
            p = FactorizeParams(seed=42, cluster=ClusterParams(m_target=256))
            if not args.apply_only:
                run_factorize("c5", inp, p, reps=2)
            lib = api.library()
            n = inp[0]
            h = api.factorize_handle(BlockedSparseMatrix.from_triplets(*inp), p)
            op = ctypes.c_void_p()
            err = lib.errbuf()
            abi.raise_for(lib.operator_create(h, 1e-12, ctypes.byref(op), err, len(err)), err)
            lib.result_free(h)
            for nrhs in (1, 20):
                v = np.random.default_rng(1).standard_normal((nrhs, n))
                out = np.zeros_like(v)
                for rep in range(3):
                    t = time.time()
                    abi.raise_for(lib.operator_apply(op, 2, nrhs, v.ctypes.data, out.ctypes.data, 0, err, len(err)),
                                  err)
                    dt = time.time() - t
                print(f"c5 apply inv_sqrt nrhs={nrhs}: {dt * 1e3:.2f} ms (host buffers)", flush=True)
            import torch  # device buffers for the device-resident apply timing
            for nrhs in (1, 20):
                dv = torch.randn(nrhs, n, dtype=torch.float64, device="cuda")
                do = torch.empty_like(dv)
                for rep in range(6):
                    torch.cuda.synchronize()
                    t = time.time()
                    abi.raise_for(lib.operator_apply(op, 2, nrhs, dv.data_ptr(), do.data_ptr(), 1, err, len(err)), err)
                    torch.cuda.synchronize()
                    dt = time.time() - t
                print(f"c5 apply inv_sqrt nrhs={nrhs}: {dt * 1e3:.3f} ms (device buffers)", flush=True)
            if args.no_pcg:
                lib.operator_free(op)
                continue
            coo, keep = abi.make_coo(*inp)
            cfg = abi.SolveConfig(1e-8, args.max_iter, args.rhs, 42)
            it = np.zeros(args.rhs, np.int32)
            cv = np.zeros(args.rhs, np.int32)
            bk = np.zeros(args.rhs, np.int32)
            tr = np.zeros((args.rhs, args.max_iter + 1))
            wall = ctypes.c_double()
            abi.raise_for(lib.solve(ctypes.byref(coo), op, ctypes.byref(cfg), it.ctypes.data_as(abi.c_i32p),
                                    cv.ctypes.data_as(abi.c_i32p), bk.ctypes.data_as(abi.c_i32p),
                                    tr.ctypes.data_as(abi.c_f64p), ctypes.byref(wall), err, len(err)), err)
            print(f"c5 pcg: rhs={args.rhs} iterations={it.tolist()} converged={int(cv.sum())} "
                  f"breakdown={int(bk.sum())} wall={wall.value:.1f} ms "
                  f"({wall.value / max(1, it.max()):.3f} ms per iteration of the batch)", flush=True)
            print("   rhs0 residuals[0:10]:", tr[0, :10].tolist(), flush=True)
            lib.operator_free(op)


if __name__ == "__main__":
    main()
