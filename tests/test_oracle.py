"""CPU: the restatement oracle (oracle/liboracle.so) is pinned bit-for-bit to
the reference compiled in place (oracle/_ref/libpmmf_ref.so) on every parity
case, and to the committed golden fixtures (tests/golden/)."""
import ctypes

import numpy as np
import pytest

import cases
import oracles
from paper_1507_04396_b200 import abi

needs_ref = pytest.mark.skipif(not oracles.available("ref"), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("name", cases.FAST)
def test_restatement_matches_reference(name):
    inp, params, part = cases.build(name)
    a = oracles.factorize("ref", inp, params, part)
    b = oracles.factorize("oracle", inp, params, part)
    oracles.assert_same(a, b)


@needs_ref
@pytest.mark.slow
@pytest.mark.parametrize("name", ["rmat14_m32", "c1_dense1024", "c2_rmat16"])
def test_restatement_matches_reference_large(name):
    inp, params, part = cases.build(name)
    oracles.assert_same(oracles.factorize("ref", inp, params, part), oracles.factorize("oracle", inp, params, part))
