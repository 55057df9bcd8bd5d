"""Seeded inputs for the comparison preconditioners and the Nystrom sketch
(solver.hpp:222-340, transform_ops.hpp:252-307), shared by the CPU pins
(restatement vs the compiled reference) and the GPU parity tests."""
import numpy as np

import cases
from cases import api


def indefinite_offdiag(n, fill=0.25, seed=11):
    """Positive diagonal, random-sign off-diagonals: IC(0) breaks down and
    restarts on A + alpha diag(A) (solver.hpp:315-333)."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n)) * (rng.random((n, n)) < fill)
    a = np.triu(a, 1)
    a = a + a.T
    a[np.diag_indices(n)] = 0.5 + rng.random(n)
    r, c = np.nonzero(a)
    return n, r.astype(np.int64), c.astype(np.int64), a[r, c]


def missing_diagonal(n=40, seed=4):
    """A zero diagonal entry at row 7 (never stored)."""
    n, r, c, v = cases.random_sym(n, 0.2, seed, shift=3.0)
    keep = ~((r == 7) & (c == 7))
    return n, r[keep], c[keep], v[keep]


def build(name):
    """Returns (input, partition or None)."""
    if name == "grid16":
        return api.workload_aniso_grid(16), None
    if name == "grid24_iso":
        return api.workload_aniso_grid(24, 1.0, 1.0), None
    if name == "rmat9":
        return api.workload_rmat(9, 16, 42), None
    if name == "dense64":
        return api.workload_dense_spd(64, 32, 42), None
    if name == "indefinite60":
        return indefinite_offdiag(60), None
    if name == "indefinite60_part":
        inp = indefinite_offdiag(60, seed=12)
        return inp, cases.shuffled_partition(60, 5)
    if name == "dups_zeros":
        return cases.with_dups_and_zeros(api.workload_aniso_grid(12)), None
    if name == "rmat9_part":
        return api.workload_rmat(9, 16, 7), cases.shuffled_partition(512, 6)
    raise KeyError(name)


NAMES = ["grid16", "grid24_iso", "rmat9", "dense64", "indefinite60", "indefinite60_part", "dups_zeros", "rmat9_part"]
