"""GPU parity at the BASELINE.json config shapes, diffed directly against the
reference compiled in place (oracle/_ref, pmmf::factorize,
factorizer.hpp:397-595) — not the restatement — on the largest sizes the CPU
reference finishes in seconds to a minute on the GPU box's host cores
(SURVEY.md §8(d) "Oracle feasibility"):

* config 4's recipe (R-MAT epv 32, m=512, c_max=10^4) at scale 14 (the
  bench's --impl reference sample) and scale 16;
* config 5 (anisotropic Poisson, m=256) at 256^2 and 512^2, plus the
  MmfOperator inv_sqrt apply (transform_ops.hpp:51-67) at 256^2;
* config 3 (RBF in 10-D, k=3, P=10, m=16) at n=2,048;
* config 2 at full size (R-MAT scale 16, epv 16, m=64).

The inputs come from the reference's own pmmf::Rng (oracle/ref_driver.cpp);
tests/test_workloads.py shows the library's generators emit the same
triplets.  Everything is compared bit-for-bit: partitions, pivot tuples,
rotation matrices, wavelet sets and order, retired diagonals, elimination
masses, residual_sq, the core.
"""
import os

import numpy as np
import pytest

import oracles
from paper_1507_04396_b200.abi import make_params

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not oracles.available("ref"), reason="oracle/_ref not built")]


def c4_params():
    return make_params(k=2, n_stages=15, eta=0.5, m_target=512, c_min=10, c_max=10000, d_max=500,
                       bypass_enabled=True, core_min=10, core_cap=4096, seed=42)


SHAPES = {
    "c4_rmat14_m512": (("rmat", 14, 32, 42, 1e-2), c4_params),
    "c4_rmat16_m512": (("rmat", 16, 32, 42, 1e-2), c4_params),
    "c5_grid256_m256": (("aniso_grid", 256, 100.0, 1.0), lambda: make_params(k=2, n_stages=15, m_target=256, seed=42)),
    "c5_grid512_m256": (("aniso_grid", 512, 100.0, 1.0), lambda: make_params(k=2, n_stages=15, m_target=256, seed=42)),
    "c3_rbf2048_k3_m16": (("rbf", 2048, 10, 0.5, 42, 1e-4),
                          lambda: make_params(k=3, n_stages=10, eta=0.5, m_target=16, c_min=10, c_max=10000,
                                              d_max=500, seed=42)),
    "c2_rmat16_m64": (("rmat", 16, 16, 42, 1e-2), lambda: make_params(m_target=64, seed=42)),
}


@pytest.fixture(scope="module", autouse=True)
def _threads():
    oracles.load("ref").lib.pmmf_ref_set_threads(os.cpu_count() or 1)


@pytest.mark.parametrize("name", list(SHAPES))
def test_factorize_matches_reference(name):
    (kind, *args), mk = SHAPES[name]
    inp = oracles.ref_workload(kind, *args)
    params = mk()
    gpu = oracles.factorize("gpu", inp, params)
    ref = oracles.factorize("ref", inp, params)
    oracles.assert_same(gpu, ref)
    assert sum(len(s.rot_indices) for s in gpu.stages) > 0


def test_operator_apply_matches_reference_c5_256():
    (kind, *args), mk = SHAPES["c5_grid256_m256"]
    inp = oracles.ref_workload(kind, *args)
    params = mk()
    vecs = np.random.default_rng(5).standard_normal((4, inp[0]))
    for mode in (0, 1, 2):
        g, gneg = oracles.operator_apply("gpu", inp, params, mode, vecs)
        r, rneg = oracles.operator_apply("ref", inp, params, mode, vecs)
        assert np.array_equal(g, r), f"mode {mode}"
        assert gneg == rneg
