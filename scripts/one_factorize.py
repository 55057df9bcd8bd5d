"""Runs one factorization of a named workload (for profiling)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_04396_b200 import api
from paper_1507_04396_b200.api import FactorizeParams, ClusterParams, BlockedSparseMatrix
c = sys.argv[1] if len(sys.argv) > 1 else "c2"
if c == "c2": inp = api.workload_rmat(16, 16, 42); p = FactorizeParams(seed=42, cluster=ClusterParams(m_target=64))
if c == "s16m512": inp = api.workload_rmat(16, 32, 42); p = FactorizeParams(seed=42, cluster=ClusterParams(m_target=512, c_max=10000))
if c == "c4": inp = api.workload_rmat(20, 32, 42); p = FactorizeParams(seed=42, cluster=ClusterParams(m_target=512, c_max=10000))
if c == "s19": inp = api.workload_rmat(19, 32, 42); p = FactorizeParams(seed=42, cluster=ClusterParams(m_target=512, c_max=10000))
if c == "s18": inp = api.workload_rmat(18, 32, 42); p = FactorizeParams(seed=42, cluster=ClusterParams(m_target=512, c_max=10000))
t = time.time(); f = api.factorize(BlockedSparseMatrix.from_triplets(*inp), p)
print(c, "wall", time.time() - t, "phases", f.phases.round(1), "launches", api.kernel_launches())
