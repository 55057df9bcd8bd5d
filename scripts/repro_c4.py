"""Repeated config-4 factorizations in one process, reporting failures and
the residual / rotation count of each (nondeterminism hunt)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_04396_b200 import api
from paper_1507_04396_b200.api import FactorizeParams, ClusterParams, BlockedSparseMatrix
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
inp = api.workload_rmat(20, 32, 42)
p = FactorizeParams(seed=42, cluster=ClusterParams(m_target=512, c_max=10000))
m = BlockedSparseMatrix.from_triplets(*inp)
for i in range(n):
    t = time.time()
    try:
        f = api.factorize(m, p)
        print("run", i, round(time.time() - t, 3), "rot", sum(len(s.rot_indices) for s in f.stages), "res", repr(f.residual_sq), flush=True)
    except Exception as e:
        print("run", i, "FAILED", e, flush=True)
