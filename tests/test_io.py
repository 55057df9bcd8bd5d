"""Input path (io.hpp:27-250) against the reference
compiled in place (oracle/_ref, pmmf_ref_* forwarding to pmmf::read_matrix_market,
read_edge_list, write_matrix_market, laplacian, symmetrize).

CPU: the text readers and the writer — same triplets (bit-exact values, same
order) or the same DataError on every file, edge cases included.
GPU: the device Laplacian and symmetrization equal the reference bit-for-bit
(its degrees and pair sums are sequential in input order)."""
import ctypes

import numpy as np
import pytest

import oracles
from paper_1507_04396_b200 import abi, api

pytestmark = pytest.mark.skipif(not oracles.available("ref"), reason="reference not built here")

MM_FILES = {
    "general_real": "%%MatrixMarket matrix coordinate real general\n% comment\n\n3 3 4\n1 1 2.5\n2 1 -1e-3\n"
                    "3 3 0x1p-3\n1 3 7\n",
    "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n4 4 4\n1 1 1.0\n2 1 -0.5\n4 2 3\n3 3 -0.0\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n3 2 3\n1 1\n3 2\n2 2\n",
    "integer_upper": "%%MatrixMarket MATRIX Coordinate Integer SYMMETRIC\n2 2 2\n1 1 4\n2 1 -2\n",
    "crlf_comments": "%%MatrixMarket matrix coordinate real general\r\n%c\r\n2 2 2\r\n% mid\r\n1 2 1.25\r\n"
                     "2 1 1.25\r\n",
    # a CRLF blank line is "\r", not empty: the reference rejects it as an entry line
    "bad_crlf_blank_line": "%%MatrixMarket matrix coordinate real general\r\n2 2 2\r\n1 2 1.25\r\n\r\n"
                           "2 1 1.25\r\n",
    "rect_extra_tokens": "%%MatrixMarket matrix coordinate real general\n2 5 2\n1 5 1e300 x\n2 1 1.000000000000000222\n",
    "empty_matrix": "%%MatrixMarket matrix coordinate real general\n0 0 0\n",
    "bad_empty": "",
    "bad_header": "%%Matrix matrix coordinate real general\n1 1 1\n1 1 1\n",
    "bad_array": "%%MatrixMarket matrix array real general\n1 1\n1\n",
    "bad_complex": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "bad_hermitian": "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n",
    "bad_size": "%%MatrixMarket matrix coordinate real general\n2 x 1\n1 1 1\n",
    "bad_negative_size": "%%MatrixMarket matrix coordinate real general\n-2 2 1\n1 1 1\n",
    "bad_eof": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n2 2 2\n",
    "bad_range": "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n",
    "bad_zero_index": "%%MatrixMarket matrix coordinate real general\n2 2 1\n0 1 1\n",
    "bad_missing_value": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",
    "bad_number": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.5q\n",
    "bad_index": "%%MatrixMarket matrix coordinate real general\n2 2 1\n+1 1 1\n",
    "bad_inf": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 inf\n",
    "bad_overflow": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1e999\n",
    "bad_single_token": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1\n",
}

EL_FILES = {
    "weighted": "# SNAP style\n10 20 0.5\n20 30\n30 10 2 # trailing comment\n\n10 10 4\n",
    "unweighted": "5 7\n7 9\n9 5\n100 5\n",
    "tabs_extra": "1\t2\t3.5\textra\n2 3\n",
    "bad_single": "1 2\n3\n",
    "bad_empty": "# nothing here\n\n",
    "bad_weight": "1 2 abc\n",
    "bad_nan": "1 2 nan\n",
    "bad_id": "1 2.0\n",
}


def _both(kind, path):
    out = []
    for lib in (api._io(), abi.IoAbi(oracles.load("ref").lib, "pmmf_ref_", device_args=False)):
        try:
            out.append(("ok", lib.read(kind, path)))
        except abi.PmmfError as e:
            out.append(("err", type(e).__name__))
    return out


def _same(a, b):
    assert a[0] == b[0], (a, b)
    if a[0] == "err":
        assert a[1] == b[1]
        return
    x, y = a[1], b[1]
    assert x[0] == y[0] and x[1] == y[1]
    for u, v in zip(x[2:5], y[2:5]):
        assert u.dtype == v.dtype and np.array_equal(u, v)
        if u.dtype == np.float64:
            assert np.array_equal(np.signbit(u), np.signbit(v))
    assert (x[5] is None) == (y[5] is None)
    if x[5] is not None:
        assert np.array_equal(x[5], y[5])


@pytest.mark.parametrize("name", sorted(MM_FILES))
def test_matrix_market_matches_reference(name, tmp_path):
    p = tmp_path / "m.mtx"
    p.write_bytes(MM_FILES[name].encode())
    ours, ref = _both("mm", str(p))
    _same(ours, ref)
    assert (ours[0] == "err") == name.startswith("bad_")


@pytest.mark.parametrize("name", sorted(EL_FILES))
def test_edge_list_matches_reference(name, tmp_path):
    p = tmp_path / "g.txt"
    p.write_bytes(EL_FILES[name].encode())
    ours, ref = _both("el", str(p))
    _same(ours, ref)
    assert (ours[0] == "err") == name.startswith("bad_")


def test_missing_files(tmp_path):
    for kind in ("mm", "el"):
        ours, ref = _both(kind, str(tmp_path / "nope"))
        assert ours == ref == ("err", "DataError") or (ours[0] == ref[0] == "err")


def test_write_matrix_market_bytes_and_round_trip(tmp_path):
    rng = np.random.default_rng(5)
    n = 300
    r = rng.integers(0, n, 2000)
    c = rng.integers(0, n, 2000)
    v = rng.standard_normal(2000) * 10.0 ** rng.integers(-300, 300, 2000)
    v[:3] = [0.0, -0.0, 1.0 / 3.0]
    a, b = tmp_path / "a.mtx", tmp_path / "b.mtx"
    api.write_matrix_market(str(a), n, n, r, c, v)
    abi.IoAbi(oracles.load("ref").lib, "pmmf_ref_", device_args=False).write_matrix_market(str(b), n, n, r, c, v)
    assert a.read_bytes() == b.read_bytes()
    rows, cols, r2, c2, v2 = api.read_matrix_market(str(a))
    assert (rows, cols) == (n, n)
    assert np.array_equal(r2, r) and np.array_equal(c2, c) and np.array_equal(v2, v)
    assert np.array_equal(np.signbit(v2), np.signbit(v))


def _ref_io():
    return abi.IoAbi(oracles.load("ref").lib, "pmmf_ref_", device_args=False)


def _random_adjacency(n, m, seed, dups=True):
    rng = np.random.default_rng(seed)
    r = rng.integers(0, n, m)
    c = rng.integers(0, n, m)
    v = rng.random(m) * 10.0 ** rng.integers(-8, 8, m)
    if dups and m >= 16:  # repeated pairs in both orientations, zeros and negative zeros
        k = m // 4
        r[:k], c[:k] = c[k:2 * k], r[k:2 * k]
        v[5:9] = [0.0, -0.0, 0.0, -0.0]
    return r, c, v


def _equal3(x, y):
    for u, w in zip(x, y):
        assert len(u) == len(w) and np.array_equal(u, w)
        if u.dtype == np.float64:
            assert np.array_equal(np.signbit(u), np.signbit(w))


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,shift", [(1, 0, 0.0), (50, 400, 0.0), (1000, 20000, 1e-2), (4096, 200000, 3.0)])
def test_gpu_laplacian_matches_reference(n, m, shift):
    r, c, v = _random_adjacency(n, m, 11 + n)
    v = np.abs(v)
    _equal3(api.laplacian(r, c, v, n, shift), _ref_io().laplacian(r, c, v, n, shift))


@pytest.mark.gpu
def test_gpu_laplacian_errors():
    r = np.array([0, 1, 5, 2]), np.array([1, 0, 1, 2])
    v = np.array([1.0, -1.0, 1.0, 1.0])
    # first offending triplet decides: negative weight (index 1) before range (index 2)
    with pytest.raises(abi.DataError, match="negative weight"):
        api.laplacian(r[0], r[1], v, 3)
    v2 = np.array([1.0, 1.0, 1.0, -1.0])
    with pytest.raises(abi.DataError, match="index out of range"):
        api.laplacian(r[0], r[1], v2, 3)
    for lib in (_ref_io(),):
        with pytest.raises(abi.DataError, match="negative weight"):
            lib.laplacian(r[0], r[1], v, 3)
        with pytest.raises(abi.DataError, match="index out of range"):
            lib.laplacian(r[0], r[1], v2, 3)


@pytest.mark.gpu
@pytest.mark.parametrize("n,m", [(1, 1), (30, 200), (1000, 50000), (100000, 400000)])
def test_gpu_symmetrize_matches_reference(n, m):
    r, c, v = _random_adjacency(n, m, 3 + m)
    v = v * np.where(np.arange(m) % 3 == 0, -1.0, 1.0)
    _equal3(api.symmetrize(r, c, v), _ref_io().symmetrize(r, c, v))


@pytest.mark.gpu
def test_gpu_edge_list_to_laplacian_pipeline(tmp_path):
    """read_edge_list -> symmetrize -> laplacian: the reference's CLI ingest
    chain, ours (device) against the reference's (host)."""
    rng = np.random.default_rng(2)
    lines = [f"{a} {b} {w:.6g}" for a, b, w in zip(rng.integers(0, 5000, 30000) * 7, rng.integers(0, 5000, 30000) * 7,
                                                   rng.random(30000))]
    p = tmp_path / "g.txt"
    p.write_text("\n".join(lines) + "\n")
    n, r, c, v, ids = api.read_edge_list(str(p))
    ref = _ref_io()
    rn, _, rr, rc, rv, rids = ref.read("el", str(p))
    assert n == rn and np.array_equal(ids, rids)
    s_ours = api.symmetrize(r, c, v)
    s_ref = ref.symmetrize(rr, rc, rv)
    _equal3(s_ours, s_ref)
    _equal3(api.laplacian(*s_ours, n, 1e-2), ref.laplacian(*s_ref, n, 1e-2))
