"""GPU MmfOperator (transform_ops.hpp:30-137) and CG harness (solver.hpp)
against the CPU oracle on the same seeded factorizations.

apply/apply_inverse/apply_inv_sqrt are bit-for-bit (same rotation
arithmetic, same core Jacobi).  CG traces use deterministic tree
reductions for the dot products instead of the reference's sequential sums
over n, so they agree to a tolerance (stated per assertion), not bitwise."""
import numpy as np
import pytest

import cases
import oracles

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["grid32_m16", "rmat12_m16", "rbf256_k3", "dense256_m2", "partitioned_input", "zero_cols_bypass"])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_apply_bitwise(name, mode):
    inp, params, part = cases.build(name)
    rng = np.random.default_rng(17)
    vecs = rng.standard_normal((5, inp[0]))
    g, gneg = oracles.operator_apply("gpu", inp, params, mode, vecs, clusters=part)
    o, oneg = oracles.operator_apply("oracle", inp, params, mode, vecs, clusters=part)
    assert gneg == oneg
    assert np.array_equal(g, o)


def test_apply_matches_reference_library():
    inp, params, part = cases.build("grid64_m16")
    vecs = np.random.default_rng(3).standard_normal((3, inp[0]))
    g, _ = oracles.operator_apply("gpu", inp, params, 2, vecs)
    r, _ = oracles.operator_apply("ref", inp, params, 2, vecs)
    assert np.array_equal(g, r)


@pytest.mark.parametrize("precondition", [True, False])
def test_cg_traces(precondition):
    inp = cases.api.workload_aniso_grid(48)
    params = cases.make_params(m_target=16, seed=42)
    gi, gc, gb, gt, _ = oracles.solve("gpu", inp, params, 1e-8, 3000, 4, 5, precondition)
    oi, oc, ob, ot, _ = oracles.solve("oracle", inp, params, 1e-8, 3000, 4, 5, precondition)
    assert np.array_equal(gc, oc) and np.array_equal(gb, ob)
    # iteration counts within 2% (rounding of the dot products differs)
    assert np.all(np.abs(gi - oi) <= np.maximum(2, 0.02 * oi)), (gi, oi)
    # the first 20 residuals agree to 1e-9 relative
    k = 20
    assert np.allclose(gt[:, :k], ot[:, :k], rtol=1e-9, atol=0)


def test_cached_blocks_reused_and_released():
    """Large device blocks stay cached between factorizations (reuse, no
    fresh mapping) and pmmf_b200_cached_bytes(release=1) hands them back."""
    from paper_1507_04396_b200 import api
    from paper_1507_04396_b200.api import BlockedSparseMatrix, ClusterParams, FactorizeParams

    inp = api.workload_rmat(16, 32, 7)
    m = BlockedSparseMatrix.from_triplets(*inp)
    p = FactorizeParams(seed=3, cluster=ClusterParams(m_target=64))
    a = api.factorize(m, p)
    cached = api.cached_device_bytes(0)
    assert cached > 0
    b = api.factorize(m, p)
    assert np.array_equal(a.core, b.core) and a.residual_sq == b.residual_sq
    assert api.cached_device_bytes(0, release=True) == 0
    assert api.cached_device_bytes(0) == 0


@pytest.mark.parametrize("name", ["rmat12_m16", "grid64_m16", "dense256_m2", "rbf512_k4", "k3_sparse"])
def test_reconstruction_error_matches_reference(name):
    """||A - Q^T H Q||_F / ||A||_F reconstructed on the GPU agrees with the
    reference's dense residual_frobenius (on its own factorization of the
    same input) within 1e-9 relative, the north-star bar, and with the
    accumulated residual."""
    import ctypes

    from paper_1507_04396_b200 import abi, api

    if not oracles.available("ref"):
        pytest.skip("reference not built")
    inp, params, part = cases.build(name)
    n, rows, cols, vals = inp
    lib, h = oracles.result_handle("gpu", inp, params, part)
    try:
        mat = api.BlockedSparseMatrix.from_triplets(n, rows, cols, vals,
                                                    api.Partition(part) if part is not None else None)
        dense = api.residual_frobenius(h, mat, "dense")
        acc = api.residual_frobenius(h, mat, "accumulated")
    finally:
        lib.result_free(h)
    rlib, rh = oracles.result_handle("ref", inp, params, part)
    try:
        coo, keep = abi.make_coo(n, rows, cols, vals, part)
        ra, rd = ctypes.c_double(), ctypes.c_double()
        err = rlib.errbuf()
        abi.raise_for(rlib.lib.pmmf_ref_residual_frobenius(rh, ctypes.byref(coo), ctypes.byref(ra), ctypes.byref(rd),
                                                           err, len(err)), err)
    finally:
        rlib.result_free(rh)
    fro = float(np.sqrt(np.sum(np.asarray(vals, np.float64) ** 2)))
    assert acc == ra.value  # bit-identical factorizations
    assert abs(dense - rd.value) <= 1e-9 * fro, (dense, rd.value, fro)
    assert abs(dense - acc) <= 1e-9 * fro, (dense, acc)
