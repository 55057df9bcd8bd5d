"""GPU: the device path raises the reference's exceptions for bad input
(factorizer.hpp:44-50, :404-408, :573-576; blocked_matrix.hpp:143-149)."""
import numpy as np
import pytest

import oracles
from paper_1507_04396_b200 import abi
from paper_1507_04396_b200.abi import make_params

pytestmark = pytest.mark.gpu


def run_both(inp, params, part=None):
    errs = []
    for which in ["gpu", "oracle"]:
        with pytest.raises(abi.PmmfError) as e:
            oracles.factorize(which, inp, params, part)
        errs.append(e.value)
    assert type(errs[0]) is type(errs[1]), errs
    return errs[0]


def sym(n=20):
    i = np.arange(n, dtype=np.int64)
    return n, np.concatenate([i, i[:-1], i[1:]]), np.concatenate([i, i[1:], i[:-1]]), np.concatenate([np.full(n, 4.0), np.full(n - 1, -1.0), np.full(n - 1, -1.0)])


def test_asymmetric_input():
    n, r, c, v = sym()
    v = v.copy()
    v[n] = -0.5
    assert isinstance(run_both((n, r, c, v), make_params()), abi.InvalidArgument)


def test_index_out_of_range():
    n, r, c, v = sym()
    r = r.copy()
    r[3] = n + 5
    assert isinstance(run_both((n, r, c, v), make_params()), abi.OutOfRange)


def test_non_finite():
    n, r, c, v = sym()
    v = v.copy()
    v[2] = np.inf
    assert isinstance(run_both((n, r, c, v), make_params()), abi.InvalidArgument)


def test_bad_params():
    inp = sym()
    assert isinstance(run_both(inp, make_params(k=9)), abi.InvalidArgument)
    assert isinstance(run_both(inp, make_params(eta=1.0)), abi.InvalidArgument)
    assert isinstance(run_both(inp, make_params(c_min=10, c_max=5)), abi.InvalidArgument)


def test_core_cap():
    inp = sym(64)
    assert isinstance(run_both(inp, make_params(n_stages=1, core_cap=8, m_target=2)), abi.NumericError)


def test_uncovered_index():
    n, r, c, v = sym()
    part = [np.arange(n - 1)]
    assert isinstance(run_both((n, r, c, v), make_params(), part), abi.OutOfRange)
