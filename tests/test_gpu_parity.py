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


@pytest.mark.parametrize("name", ["rmat12_m16", "grid64_m16", "dense256_m2", "rbf512_k4", "zero_cols_bypass",
                                  "partitioned_input", "k3_sparse"])
def test_small_batches_and_chunks(name, monkeypatch):
    """Force many cluster batches in the row pass and tiny transpose chunks
    (the paths config 4 takes for memory) — still bit-exact."""
    monkeypatch.setenv("PMMF_B200_BATCH_NNZ", "2000")
    monkeypatch.setenv("PMMF_B200_CHUNK_NNZ", "3000")
    inp, params, part = cases.build(name)
    oracles.assert_same(oracles.factorize("gpu", inp, params, part), oracles.factorize("oracle", inp, params, part))


@pytest.mark.parametrize("name", ["rmat12_m16", "grid64_m16", "dense256_m2", "rbf512_k4", "zero_cols_bypass",
                                  "partitioned_input", "k3_sparse"])
@pytest.mark.parametrize("div", ["1e9", "3"])
def test_dense_scoring_path(name, div, monkeypatch):
    """Route every (div=1e9) or only the heaviest (div=3) pool columns through
    the dense-gather scorer (hub columns on config 4) — still bit-exact."""
    monkeypatch.setenv("PMMF_B200_DENSE_DIV", div)
    inp, params, part = cases.build(name)
    oracles.assert_same(oracles.factorize("gpu", inp, params, part), oracles.factorize("oracle", inp, params, part))


@pytest.mark.parametrize("name", ["rmat12_m16", "grid64_m16", "dense256_m2", "rbf512_k4", "zero_cols_bypass",
                                  "partitioned_input", "k3_sparse"])
@pytest.mark.parametrize("csize", ["2", "4", "16"])
def test_cluster_search_path(name, csize, monkeypatch):
    """Every cluster through the thread-block-cluster search kernel (the
    large-cluster path on config 4), 2- and 16-CTA clusters — still bit-exact."""
    monkeypatch.setenv("PMMF_B200_SEARCH_BIG_C", "2")
    monkeypatch.setenv("PMMF_B200_SEARCH_CSIZE", "16")
    monkeypatch.setenv("PMMF_B200_SEARCH_FORCE_W", csize)
    inp, params, part = cases.build(name)
    oracles.assert_same(oracles.factorize("gpu", inp, params, part), oracles.factorize("oracle", inp, params, part))


@pytest.mark.parametrize("name", ["rmat12_m16", "grid64_m16", "dense256_m2", "rbf256_k3", "rbf512_k4",
                                  "zero_cols_bypass", "partitioned_input", "k3_sparse", "dups_and_zeros",
                                  "undersize_repair", "c1_dense1024"])
@pytest.mark.parametrize("ratio", ["1e30", "0"])
def test_gram_paths(name, ratio, monkeypatch):
    """Every cluster's Gram through the dense sequential SYRK (ratio=1e30:
    zero-filled panels, exact-zero products inserted) or through the sparse
    row-run path (ratio=0) — both bit-exact against the oracle."""
    monkeypatch.setenv("PMMF_B200_GRAM_DENSE_RATIO", ratio)
    inp, params, part = cases.build(name)
    oracles.assert_same(oracles.factorize("gpu", inp, params, part), oracles.factorize("oracle", inp, params, part))


@pytest.mark.parametrize("name", ["rmat12_m16", "grid64_m16", "dense256_m2", "rbf256_k3", "rbf512_k4",
                                  "zero_cols_bypass", "partitioned_input", "oversize_recursion",
                                  "undersize_repair", "c1_dense1024"])
@pytest.mark.parametrize("gemm", ["1", "0"])
def test_score_gemm_path(name, gemm, monkeypatch):
    """Clustering scores through the dense GEMM scorer (gemm=1: zero-filled
    panels, two-level block sums per thread) or never through it (gemm=0,
    the sparse row-inverted scorer on dense inputs) — bit-exact either way,
    including the orphan re-scoring table (rows mode) of undersize repair."""
    monkeypatch.setenv("PMMF_B200_SCORE_GEMM", gemm)
    inp, params, part = cases.build(name)
    oracles.assert_same(oracles.factorize("gpu", inp, params, part), oracles.factorize("oracle", inp, params, part))


@pytest.mark.parametrize("name", ["rmat12_m16", "grid64_m16", "dense256_m2", "rbf512_k4", "k3_sparse",
                                  "partitioned_input"])
@pytest.mark.parametrize("batch", ["0", "2000"])
def test_level_loop_path(name, batch, monkeypatch):
    """The opt-in persistent level loop (one cooperative launch per batch,
    partitions ordered by a decoupled look-back) — bit-exact, also with many
    batches and arena compactions."""
    monkeypatch.setenv("PMMF_B200_LEVEL_LOOP", "1")
    if batch != "0":
        monkeypatch.setenv("PMMF_B200_BATCH_NNZ", batch)
        monkeypatch.setenv("PMMF_B200_MERGE_CHUNK", "32")
    inp, params, part = cases.build(name)
    oracles.assert_same(oracles.factorize("gpu", inp, params, part), oracles.factorize("oracle", inp, params, part))


@pytest.mark.parametrize("name", ["rmat12_m16", "grid64_m16", "dense256_m2", "rbf512_k4", "zero_cols_bypass",
                                  "partitioned_input", "undersize_repair", "oversize_recursion"])
def test_long_column_norms(name, monkeypatch):
    """Every column longer than 8 entries through the CTA-per-column norm
    kernel (hub columns on config 4) — still bit-exact."""
    monkeypatch.setenv("PMMF_B200_NORM_LONG", "8")
    inp, params, part = cases.build(name)
    oracles.assert_same(oracles.factorize("gpu", inp, params, part), oracles.factorize("oracle", inp, params, part))


@pytest.mark.parametrize("name", ["rmat12_m16", "grid64_m16", "dense256_m2", "rbf512_k4", "k3_sparse",
                                  "partitioned_input"])
@pytest.mark.parametrize("below", ["8", "64"])
def test_level_loop_hybrid(name, below, monkeypatch):
    """The per-level chain for a batch's large levels, then one level-loop
    launch for its tail of small levels — bit-exact, with compactions."""
    monkeypatch.setenv("PMMF_B200_LOOP_BELOW", below)
    monkeypatch.setenv("PMMF_B200_BATCH_NNZ", "5000")
    inp, params, part = cases.build(name)
    oracles.assert_same(oracles.factorize("gpu", inp, params, part), oracles.factorize("oracle", inp, params, part))


@pytest.mark.parametrize("name", ["rmat12_m16", "grid64_m16", "dense256_m2", "partitioned_input",
                                  "undersize_repair", "oversize_recursion"])
@pytest.mark.parametrize("hook", ["chunk32", "merge2_off", "alloc_unfused", "chunk32_alloc_unfused",
                                  "gram_pipe0", "gram_pipe1", "gram_pipe2", "fine_off", "fine_32_8192"])
def test_rotation_stream_variants(name, hook, monkeypatch):
    """The k = 2 ring merge kernel with every rotation cut into 32-row
    partitions (multi-partition count pass + allocation by the last counting
    warp on small inputs), its fallbacks (generic merge kernel, separate
    allocation launch) and the sparse Gram owner kernel variants — bit-exact."""
    if "chunk32" in hook:
        monkeypatch.setenv("PMMF_B200_MERGE_CHUNK", "32")
        monkeypatch.setenv("PMMF_B200_BATCH_NNZ", "4000")
    if hook == "merge2_off":
        monkeypatch.setenv("PMMF_B200_MERGE2", "0")
        monkeypatch.setenv("PMMF_B200_MERGE_CHUNK", "32")
    if "alloc_unfused" in hook:
        monkeypatch.setenv("PMMF_B200_FUSED_ALLOC", "0")
    if hook == "fine_off":  # one partition size for every level
        monkeypatch.setenv("PMMF_B200_FINE_LEVELS", "0")
    if hook == "fine_32_8192":  # every level below 8192 partitions cut into 32-row partitions
        monkeypatch.setenv("PMMF_B200_FINE_CHUNK", "32")
        monkeypatch.setenv("PMMF_B200_FINE_ITEMS", "8192")
        monkeypatch.setenv("PMMF_B200_BATCH_NNZ", "4000")
    if hook.startswith("gram_pipe"):
        monkeypatch.setenv("PMMF_B200_GRAM_PIPE", hook[-1])
        monkeypatch.setenv("PMMF_B200_GRAM_DENSE_RATIO", "0")  # sparse Gram for every cluster
    inp, params, part = cases.build(name)
    oracles.assert_same(oracles.factorize("gpu", inp, params, part), oracles.factorize("oracle", inp, params, part))
