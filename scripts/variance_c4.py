"""Step-variance diagnostic: N traced config-4 factorizations back to back
(PMMF_B200_TRACE sub-phase timings on stderr, a marker line per step)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_04396_b200 import api
from paper_1507_04396_b200.api import FactorizeParams, ClusterParams, BlockedSparseMatrix
inp = api.workload_rmat(20, 32, 42)
p = FactorizeParams(seed=42, cluster=ClusterParams(m_target=512, c_max=10000))
m = BlockedSparseMatrix.from_triplets(*inp)
for _ in range(2):
    api.factorize(m, p)
os.environ["PMMF_B200_TRACE"] = "1"
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
    t = time.time(); f = api.factorize(m, p)
    print(f"=== step {i} wall {1e3 * (time.time() - t):.1f} phases {f.phases.round(1)}", file=sys.stderr, flush=True)
