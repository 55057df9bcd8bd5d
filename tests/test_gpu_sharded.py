"""Sharded factorization: the clusters of every stage split
over W ranks (shard.cuh).  On one GPU the ranks run as `virtual` ranks, one
after another in this process, with the exchanges as shared buffers; the
result must equal the CPU oracle bit-for-bit for every W — the decomposition
changes which GPU computes an entry, never how.  A one-rank NCCL
communicator runs the NCCL exchange code itself (self-broadcasts)."""
import numpy as np
import pytest

import cases
import oracles
from paper_1507_04396_b200 import api

pytestmark = pytest.mark.gpu

NAMES = ["rmat12_m16", "grid64_m16", "dense256_m2", "rbf512_k4", "zero_cols_bypass", "partitioned_input",
         "k3_sparse", "undersize_repair", "oversize_recursion", "c1_dense1024"]


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("world", [2, 3, 8])
def test_virtual_ranks_match_oracle(name, world):
    inp, params, part = cases.build(name)
    comm = api.Communicator(world, virtual=True)
    try:
        gpu = oracles.factorize("gpu", inp, params, part, comm=comm)
    finally:
        comm.close()
    oracles.assert_same(gpu, oracles.factorize("oracle", inp, params, part))


@pytest.mark.parametrize("name", ["rmat12_m16", "grid64_m16", "k3_sparse"])
def test_virtual_ranks_small_batches(name, monkeypatch):
    """Sharded slabs through many row-pass batches and tiny transpose chunks."""
    monkeypatch.setenv("PMMF_B200_BATCH_NNZ", "2000")
    monkeypatch.setenv("PMMF_B200_CHUNK_NNZ", "3000")
    inp, params, part = cases.build(name)
    comm = api.Communicator(4, virtual=True)
    try:
        gpu = oracles.factorize("gpu", inp, params, part, comm=comm)
    finally:
        comm.close()
    oracles.assert_same(gpu, oracles.factorize("oracle", inp, params, part))


@pytest.mark.parametrize("name", ["rmat12_m16", "dense256_m2", "zero_cols_bypass"])
def test_nccl_one_rank_exchanges(name):
    """The NCCL path (grouped in-place broadcasts of the rotation slots,
    masses and column slabs) on a one-rank communicator."""
    inp, params, part = cases.build(name)
    comm = api.Communicator(1, 0, 0)
    try:
        gpu = oracles.factorize("gpu", inp, params, part, comm=comm)
    finally:
        comm.close()
    oracles.assert_same(gpu, oracles.factorize("oracle", inp, params, part))


def test_sharded_rmat16_full():
    """C2 (R-MAT n = 65,536, m = 64) on 4 virtual ranks equals the one-GPU path."""
    inp, params, part = cases.build("c2_rmat16")
    comm = api.Communicator(4, virtual=True)
    try:
        sharded = oracles.factorize("gpu", inp, params, part, comm=comm)
    finally:
        comm.close()
    oracles.assert_same(sharded, oracles.factorize("gpu", inp, params, part))


@pytest.mark.parametrize("name", ["rmat14_m32", "c1_dense1024"])
@pytest.mark.parametrize("world", [5, 16])
def test_virtual_ranks_larger(name, world):
    """More ranks than most stages have large clusters, uneven splits."""
    inp, params, part = cases.build(name)
    comm = api.Communicator(world, virtual=True)
    try:
        gpu = oracles.factorize("gpu", inp, params, part, comm=comm)
    finally:
        comm.close()
    oracles.assert_same(gpu, oracles.factorize("oracle", inp, params, part))


@pytest.mark.parametrize("name", ["rmat12_m16", "k3_sparse", "grid64_m16"])
@pytest.mark.parametrize("env", [
    {"PMMF_B200_SEARCH_BIG_C": "2", "PMMF_B200_SEARCH_CSIZE": "16", "PMMF_B200_SEARCH_FORCE_W": "4"},
    {"PMMF_B200_DENSE_DIV": "3"},
    {"PMMF_B200_GRAM_DENSE_RATIO": "1e30"},
    {"PMMF_B200_SCORE_GEMM": "1"},
], ids=["cluster_search", "dense_scoring", "dense_gram", "gemm_scorer"])
def test_virtual_ranks_alternative_paths(name, env, monkeypatch):
    """The sharded stage loop over every alternative kernel path (the sharded
    scorer only splits the sparse scorer; the GEMM scorer stays whole)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    inp, params, part = cases.build(name)
    comm = api.Communicator(3, virtual=True)
    try:
        gpu = oracles.factorize("gpu", inp, params, part, comm=comm)
    finally:
        comm.close()
    oracles.assert_same(gpu, oracles.factorize("oracle", inp, params, part))


@pytest.mark.parametrize("name", ["grid64_m16", "rmat12_m16", "rbf256_k3", "partitioned_input"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_operator_apply(name, world):
    """MmfOperator apply sharded by apply group per stage (virtual ranks):
    bit-identical to the one-GPU apply in every mode."""
    inp, params, part = cases.build(name)
    f = oracles.factorize("gpu", inp, params, part)
    op = api.MmfOperator(f)
    comm = api.Communicator(world, virtual=True)
    try:
        x = np.random.default_rng(4).standard_normal((5, inp[0]))
        for mode in (0, 1, 2):
            assert np.array_equal(op.apply_sharded(mode, x, comm), op.apply(mode, x))
    finally:
        comm.close()
        op.close()


def test_sharded_operator_apply_nccl_one_rank():
    inp, params, part = cases.build("grid64_m16")
    f = oracles.factorize("gpu", inp, params, part)
    op = api.MmfOperator(f)
    comm = api.Communicator(1, 0, 0)
    try:
        x = np.random.default_rng(5).standard_normal((3, inp[0]))
        assert np.array_equal(op.apply_sharded(2, x, comm), op.apply(2, x))
    finally:
        comm.close()
        op.close()
