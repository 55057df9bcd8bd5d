"""Dependency-level statistics of a factorization's rotations per stage and
cluster (how deep the MMF apply's level chains are)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1507_04396_b200 import api
from paper_1507_04396_b200.api import BlockedSparseMatrix, ClusterParams, FactorizeParams

c = sys.argv[1] if len(sys.argv) > 1 else "c5"
if c == "c5":
    inp = api.workload_aniso_grid(1024)
    p = FactorizeParams(seed=42, cluster=ClusterParams(m_target=256))
elif c == "c4":
    inp = api.workload_rmat(20, 32, 42)
    p = FactorizeParams(seed=42, cluster=ClusterParams(m_target=512, c_max=10000))
f = api.factorize(BlockedSparseMatrix.from_triplets(*inp), p)
n = inp[0]
for si, st in enumerate(f.stages[:6]):
    idx = st.rot_indices
    q = st.rot_matrices
    ident = np.all(q.reshape(len(q), -1) == np.array([1.0, -0.0, 0.0, 1.0]), axis=1) if len(q) else np.zeros(0, bool)
    last = np.zeros(n, np.int32)
    lv = np.zeros(len(idx), np.int32)
    for t in range(len(idx)):
        if ident[t]:
            continue
        a, b = idx[t]
        l = max(last[a], last[b]) + 1
        last[a] = l
        last[b] = l
        lv[t] = l
    off = st.cluster_offsets
    mem = st.members
    cl = np.full(n, -1, np.int64)
    for u in range(len(off) - 1):
        cl[mem[off[u]:off[u + 1]]] = u
    cu = cl[idx[:, 0]] if len(idx) else np.zeros(0, np.int64)
    nu = len(off) - 1
    maxl = np.zeros(nu, np.int64)
    np.maximum.at(maxl, cu, lv)
    cnt = np.bincount(cu, minlength=nu)
    sizes = np.diff(off)
    print(f"stage {si + 1}: {len(idx)} rotations ({int(ident.sum())} identity), clusters {nu}, "
          f"size max {sizes.max()} mean {sizes.mean():.0f}; levels per cluster max {maxl.max()} "
          f"mean {maxl.mean():.1f} median {np.median(maxl):.0f}; rotations/level mean "
          f"{(cnt / np.maximum(maxl, 1)).mean():.1f}", flush=True)
