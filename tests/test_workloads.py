"""CPU: the seeded input recipes (csrc/recipes.hpp) emit the
same triplets on the library's generator (libpmmf_b200.so, rng.cuh) and on
the reference's pmmf::Rng (oracle/_ref, rng.hpp) — the bench's reference arm
builds its input from the latter without loading libpmmf_b200.so."""
import numpy as np
import pytest

import oracles
from paper_1507_04396_b200 import api

needs_ref = pytest.mark.skipif(not oracles.available("ref"), reason="oracle/_ref not built")

CASES = {
    "rmat12_epv32": (lambda: api.workload_rmat(12, 32, 42, 1e-2), ("rmat", 12, 32, 42, 1e-2)),
    "rmat10_epv16_s7": (lambda: api.workload_rmat(10, 16, 7, 1e-2), ("rmat", 10, 16, 7, 1e-2)),
    "dense_spd128": (lambda: api.workload_dense_spd(128, 32, 42), ("dense_spd", 128, 32, 42, 1e-3)),
    "rbf200": (lambda: api.workload_rbf(200, seed=42), ("rbf", 200, 10, 0.5, 42, 1e-4)),
    "grid40": (lambda: api.workload_aniso_grid(40), ("aniso_grid", 40, 100.0, 1.0)),
}


@needs_ref
@pytest.mark.parametrize("name", list(CASES))
def test_recipe_same_on_reference_rng(name):
    ours, (kind, *args) = CASES[name]
    a = ours()
    b = oracles.ref_workload(kind, *args)
    assert a[0] == b[0]
    for x, y in zip(a[1:], b[1:]):
        assert x.dtype == y.dtype and np.array_equal(x, y)


@needs_ref
def test_rmat_known_nnz():
    """C2 (scale 16, epv 16, seed 42) has nnz = 1,020,912."""
    n, r, c, v = oracles.ref_workload("rmat", 16, 16, 42, 1e-2)
    assert n == 65536 and len(v) == 1020912
