import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1507_04396_b200 import api
from paper_1507_04396_b200.api import FactorizeParams, ClusterParams, BlockedSparseMatrix
cfgs = sys.argv[1:] or ["c2", "s18", "c4"]
for c in cfgs:
    t = time.time()
    if c == "c2": inp = api.workload_rmat(16, 16, 42); p = FactorizeParams(seed=42, cluster=ClusterParams(m_target=64))
    if c == "s18": inp = api.workload_rmat(18, 32, 42); p = FactorizeParams(seed=42, cluster=ClusterParams(m_target=512, c_max=10000))
    if c == "c4": inp = api.workload_rmat(20, 32, 42); p = FactorizeParams(seed=42, cluster=ClusterParams(m_target=512, c_max=10000))
    if c == "c5": inp = api.workload_aniso_grid(1024); p = FactorizeParams(seed=42, cluster=ClusterParams(m_target=256))
    gen = time.time() - t
    m = BlockedSparseMatrix.from_triplets(*inp)
    for rep in range(2):
        t = time.time(); f = api.factorize(m, p); wall = time.time() - t
        rots = sum(len(s.rot_indices) for s in f.stages)
        print(f"{c}: n={inp[0]} nnz={len(inp[1])} gen={gen:.1f}s wall={wall:.3f}s rot={rots} rot/s={rots/wall:.0f} stages={len(f.stages)} resid={f.residual_sq:.6e}", flush=True)
        print("   phases ms (clust,gram,search,apply,reblock,total):", np.round(f.phases, 1), flush=True)
    for row in f.stage_info: print("   ", row.tolist())
