"""Three back-to-back C4 factorizations in one process (pool warm-up study); trace on runs >= 1."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_04396_b200 import api
from paper_1507_04396_b200.api import FactorizeParams, ClusterParams, BlockedSparseMatrix
inp = api.workload_rmat(20, 32, 42)
p = FactorizeParams(seed=42, cluster=ClusterParams(m_target=512, c_max=10000))
m = BlockedSparseMatrix.from_triplets(*inp)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    if i >= 0: os.environ["PMMF_B200_TRACE"] = "1"
    t = time.time(); f = api.factorize(m, p); print("run", i, round(time.time() - t, 3), f.phases.round(0), flush=True)
