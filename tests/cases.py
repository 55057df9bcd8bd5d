"""Seeded parity cases shared by the CPU oracle tests and the GPU parity tests.

Each case is (name, input builder, FactorizeParams builder, partition) at a
size the CPU oracle finishes in seconds.  Inputs come from the workload
generators of libpmmf_b200.so (SURVEY.md §8(d) recipes) or are constructed
here for edge cases the reference's spec names.
"""
import numpy as np

from paper_1507_04396_b200 import api
from paper_1507_04396_b200.abi import make_params


def diag_matrix(n, seed=3):
    rng = np.random.default_rng(seed)
    d = rng.uniform(0.5, 2.0, n)
    i = np.arange(n, dtype=np.int64)
    return n, i, i.copy(), d


def random_sym(n, fill, seed, shift=0.0, zero_cols=()):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n)) * (rng.random((n, n)) < fill)
    a = np.triu(a)
    a = a + a.T
    a[np.diag_indices(n)] += shift
    for z in zero_cols:
        a[z, :] = 0.0
        a[:, z] = 0.0
    r, c = np.nonzero(a)
    return n, r.astype(np.int64), c.astype(np.int64), a[r, c]


def with_dups_and_zeros(inp, seed=5):
    """Split some values into duplicate triplets and add explicit zeros
    (from_triplets sums duplicates in input order, blocked_matrix.hpp:138-156)."""
    n, r, c, v = inp
    rng = np.random.default_rng(seed)
    pick = rng.random(len(v)) < 0.2
    r2, c2, v2 = r[pick], c[pick], v[pick] * 0.25
    v = v.copy()
    v[pick] = v[pick] * 0.75
    zr = rng.integers(0, n, 20)
    zc = rng.integers(0, n, 20)
    rr = np.concatenate([r, r2, zr, zc])
    cc = np.concatenate([c, c2, zc, zr])
    vv = np.concatenate([v, v2, np.zeros(40)])
    return n, rr, cc, vv


def shuffled_partition(n, parts, seed=7):
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)
    return [perm[i::parts] for i in range(parts)]


def build(name):
    """Returns (input, params, partition or None)."""
    if name == "rmat10_m8":
        return api.workload_rmat(10, 16, 42), make_params(m_target=8, seed=42), None
    if name == "rmat12_m16":
        return api.workload_rmat(12, 16, 42), make_params(m_target=16, seed=42), None
    if name == "rmat13_m64":
        return api.workload_rmat(13, 16, 7), make_params(m_target=64, seed=7), None
    if name == "rmat14_m32":
        return api.workload_rmat(14, 16, 42), make_params(m_target=32, seed=42), None
    if name == "grid32_m16":
        return api.workload_aniso_grid(32), make_params(m_target=16, seed=1), None
    if name == "grid64_m16":
        return api.workload_aniso_grid(64), make_params(m_target=16, seed=42), None
    if name == "dense256_m2":
        return api.workload_dense_spd(256, 64, 42), make_params(m_target=2, n_stages=8, seed=42), None
    if name == "c1_dense1024":
        return api.workload_dense_spd(1024, 256, 42), make_params(m_target=2, n_stages=8, seed=42), None
    if name == "rbf256_k3":
        return api.workload_rbf(256, seed=42), make_params(k=3, m_target=4, n_stages=10, c_max=10000, seed=42), None
    if name == "rbf512_k4":
        return api.workload_rbf(512, seed=42), make_params(k=4, m_target=4, n_stages=10, c_max=10000, seed=42), None
    if name == "c2_rmat16":
        return api.workload_rmat(16, 16, 42), make_params(m_target=64, seed=42), None
    if name == "diag64":
        return diag_matrix(64), make_params(m_target=4, seed=1), None
    if name == "trivial8":
        return random_sym(8, 0.5, 11, shift=4.0), make_params(m_target=2, seed=1), None
    if name == "zero_cols_bypass":
        return random_sym(120, 0.08, 12, shift=1.0, zero_cols=(3, 17, 50, 51, 99)), make_params(m_target=4, seed=3), None
    if name == "zero_cols_nobypass":
        return (random_sym(120, 0.08, 12, shift=1.0, zero_cols=(3, 17, 50, 51, 99)),
                make_params(m_target=4, bypass_enabled=False, seed=3), None)
    if name == "partitioned_input":
        inp = random_sym(200, 0.05, 13, shift=2.0)
        return inp, make_params(m_target=6, seed=9), shuffled_partition(200, 5)
    if name == "dups_and_zeros":
        return with_dups_and_zeros(random_sym(150, 0.06, 14, shift=1.0)), make_params(m_target=5, seed=4), None
    if name == "oversize_recursion":
        return api.workload_rmat(11, 16, 3), make_params(m_target=2, c_max=300, c_min=5, seed=5), None
    if name == "undersize_repair":
        return api.workload_rmat(10, 8, 9), make_params(m_target=40, c_min=30, seed=6), None
    if name == "k3_sparse":
        return api.workload_rmat(11, 16, 8), make_params(k=3, m_target=8, seed=8), None
    if name == "eta_0p3_core20":
        return api.workload_aniso_grid(40, 1.0, 1.0), make_params(m_target=8, eta=0.3, core_min=20, seed=2), None
    raise KeyError(name)


FAST = [
    "rmat10_m8", "rmat12_m16", "grid32_m16", "grid64_m16", "dense256_m2", "rbf256_k3", "rbf512_k4",
    "diag64", "trivial8", "zero_cols_bypass", "zero_cols_nobypass", "partitioned_input", "dups_and_zeros",
    "oversize_recursion", "undersize_repair", "k3_sparse", "eta_0p3_core20", "rmat13_m64",
]
SLOW = ["rmat14_m32", "c1_dense1024", "c2_rmat16"]
