"""Warm factorization, then one traced factorization (PMMF_B200_TRACE sub-phase
timings on stderr) of config 4 (or the workload named in argv[1])."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_04396_b200 import api
from paper_1507_04396_b200.api import FactorizeParams, ClusterParams, BlockedSparseMatrix
c = sys.argv[1] if len(sys.argv) > 1 else "c4"
if c == "c4": inp = api.workload_rmat(20, 32, 42); p = FactorizeParams(seed=42, cluster=ClusterParams(m_target=512, c_max=10000))
if c == "c5": inp = api.workload_aniso_grid(1024); p = FactorizeParams(seed=42, cluster=ClusterParams(m_target=256))
m = BlockedSparseMatrix.from_triplets(*inp)
for _ in range(int(os.environ.get("WARM", "1"))):
    f = api.factorize(m, p)
os.environ["PMMF_B200_TRACE"] = "1"
t = time.time(); f = api.factorize(m, p)
print(c, "wall", time.time() - t, "phases", f.phases.round(1), file=sys.stderr)
