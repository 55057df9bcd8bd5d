"""GPU parity: every factorization through libpmmf_b200.so (the C-ABI, sm_100a
kernels) must equal the CPU oracle bit-for-bit — partitions, pivot tuples,
rotation matrices, wavelet sets and their order, retired diagonals, the core
and residual_sq (SURVEY.md §8(c) parity contract, no near-ties needed on these
cases)."""
import numpy as np
import pytest

import cases
import oracles

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", cases.FAST + cases.SLOW)
def test_factorize_matches_oracle(name):
    inp, params, part = cases.build(name)
    gpu = oracles.factorize("gpu", inp, params, part)
    ref = oracles.factorize("oracle", inp, params, part)
    oracles.assert_same(gpu, ref)
