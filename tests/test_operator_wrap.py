"""MmfOperator(shared_ptr<const MmfFactorization>, zero_threshold)
(transform_ops.hpp:32-41) on the GPU: a factorization made elsewhere — here
the reference's own pmmf::factorize (oracle/_ref) — is wrapped without
refactorizing (pmmf_b200_result_create / _add_stage / _set_core) and its
applies equal the reference MmfOperator's bit for bit.  Corrupt
factorizations are rejected as DataError on the host, before any device
work (CPU tests)."""
import copy

import numpy as np
import pytest

import cases
import oracles
from paper_1507_04396_b200 import abi, api

needs_ref = pytest.mark.skipif(not oracles.available("ref"), reason="oracle/_ref not built")


def _ref_flat(name):
    inp, params, part = cases.build(name)
    return inp, params, part, oracles.factorize("ref", inp, params, part)


@needs_ref
def test_handle_round_trip_cpu():
    """Builder -> accessors reproduce the factorization exactly (host only)."""
    _, params, _, f = _ref_flat("rmat10_m8")
    lib = api.library()
    h = api.result_handle_from(f, params)
    try:
        oracles.assert_same(lib.read_result(h), f)
    finally:
        lib.result_free(h)


@needs_ref
@pytest.mark.parametrize("what", ["rot", "member", "elim", "core", "diag", "k"])
def test_corrupt_factorization_rejected(what):
    _, params, _, f = _ref_flat("rmat10_m8")
    g = copy.deepcopy(f)
    st = g.stages[0]
    if what == "rot":
        st.rot_indices = st.rot_indices.copy()
        st.rot_indices[0, 0] = g.n + 3
    elif what == "member":
        st.members = st.members.copy()
        st.members[0] = -1
    elif what == "elim":
        st.elim_index = st.elim_index.copy()
        st.elim_index[0] = g.n
    elif what == "core":
        g.core_indices = g.core_indices.copy()
        g.core_indices[0] = 1 << 40
    elif what == "diag":
        g.diag_index = g.diag_index.copy()
        g.diag_index[-1] = g.n
    elif what == "k":
        params = abi.make_params(k=9)
        g.k = 9
    with pytest.raises(abi.DataError):
        h = api.result_handle_from(g, params)
        api.library().result_free(h)


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("name", ["rmat12_m16", "grid64_m16", "rbf512_k4", "zero_cols_bypass"])
def test_operator_wraps_reference_factorization(name):
    inp, params, part, f = _ref_flat(name)
    op = api.MmfOperator(f)
    assert op.dim() == inp[0] and op.factorization() is f
    vecs = np.random.default_rng(11).standard_normal((3, inp[0]))
    for mode in (api.MmfOperator.Mode.forward, api.MmfOperator.Mode.inverse, api.MmfOperator.Mode.inv_sqrt):
        r, rneg = oracles.operator_apply("ref", inp, params, mode, vecs, clusters=part)
        assert np.array_equal(op.apply(mode, vecs), r), mode
        assert np.array_equal(op.apply(mode, vecs[0]), r[0]), mode
        assert op.inv_sqrt_zeroed_negatives() == rneg
    op.close()


@needs_ref
@pytest.mark.gpu
def test_operator_device_tensors():
    import torch

    inp, params, part, f = _ref_flat("rmat12_m16")
    op = api.MmfOperator(f)
    vecs = np.random.default_rng(12).standard_normal((5, inp[0]))
    host = op.apply(op.Mode.inv_sqrt, vecs)
    dev = op.apply(op.Mode.inv_sqrt, torch.from_numpy(vecs).cuda())
    assert np.array_equal(dev.cpu().numpy(), host)
    with pytest.raises(ValueError):
        op.apply(op.Mode.forward, torch.zeros(3, inp[0], dtype=torch.float32, device="cuda"))


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("core_min", [10, 40, 100, 300])
def test_core_eigensystem_on_device(core_min):
    """The core's jacobi_eigensystem (dense.hpp:191-199) runs on the device:
    shared-memory tiles up to g = 48, global scratch above; the inverse and
    inv_sqrt applies (which go through the eigenvectors and f(lambda)) equal
    the reference's bit for bit."""
    inp, params, part = cases.build("rmat12_m16")
    params = abi.make_params(m_target=16, seed=42, core_min=core_min)
    f = oracles.factorize("ref", inp, params, part)
    assert len(f.core_indices) >= min(core_min, inp[0])
    op = api.MmfOperator(f)
    vecs = np.random.default_rng(13).standard_normal((2, inp[0]))
    for mode in (1, 2):
        r, rneg = oracles.operator_apply("ref", inp, params, mode, vecs, clusters=part)
        assert np.array_equal(op.apply(mode, vecs), r), mode
        assert op.inv_sqrt_zeroed_negatives() == rneg
