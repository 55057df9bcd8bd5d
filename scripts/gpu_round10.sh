cd $GRAFT_REPO_ROOT
cat > /tmp/two.py <<'PY'
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_1507_04396_b200 import api
from paper_1507_04396_b200.api import FactorizeParams, ClusterParams, BlockedSparseMatrix
inp = api.workload_rmat(20, 32, 42)
p = FactorizeParams(seed=42, cluster=ClusterParams(m_target=512, c_max=10000))
m = BlockedSparseMatrix.from_triplets(*inp)
for i in range(3):
    if i >= 1: os.environ["PMMF_B200_TRACE"] = "1"
    t = time.time(); f = api.factorize(m, p); print("run", i, time.time() - t, f.phases.round(0), flush=True)
PY
timeout 600 python /tmp/two.py 2>&1 | grep -E "run |apply\.|stage [12]: (gram|apply)" | head -60
