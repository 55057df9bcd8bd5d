"""Factorization container: the reference's JSON
schema of save_factorization / load_factorization (serialize.hpp:25-183),
written and read by libpmmf_b200.so without a JSON library.

CPU tests: factorizations of the CPU oracle are written by a Python
restatement of factorization_to_json (serialize.hpp:61-110, below), loaded
through the C-ABI and must come back bit-for-bit; the library's own writer
must produce the same JSON document.  GPU test: a GPU factorization saved
and reloaded drives MmfOperator to the same bits as the original."""
import ctypes
import json
import os

import numpy as np
import pytest

import cases
import oracles
from paper_1507_04396_b200 import abi, api


def reference_json(f, p):
    """serialize.hpp:61-110 in Python (key names, nesting, row-major q/core)."""
    return {
        "format": "pmmf-factorization",
        "version": 1,
        "n": int(f.n),
        "residual_sq": float(f.residual_sq),
        "active_history": [int(x) for x in f.active_history],
        "params": {"k": p.k, "n_stages": p.n_stages, "eta": p.eta, "core_min": p.core_min, "core_cap": p.core_cap,
                   "seed": p.seed,
                   "cluster": {"m_target": p.m_target, "c_min": p.c_min, "c_max": p.c_max, "d_max": p.d_max,
                               "bypass": bool(p.bypass_enabled), "seed": p.cluster_seed}},
        "stages": [{
            "partition": [[int(x) for x in c] for c in st.clusters()],
            "bypassed": [int(x) for x in st.bypassed],
            "rotations": [{"i": [int(x) for x in st.rot_indices[t]],
                           "q": [float(x) for x in st.rot_matrices[t].reshape(-1)]}
                          for t in range(len(st.rot_indices))],
            "eliminated": [{"i": int(i), "d": float(d), "m": float(m)}
                           for i, d, m in zip(st.elim_index, st.elim_diagonal, st.elim_off_mass_sq)],
        } for st in f.stages],
        "core": {"indices": [int(x) for x in f.core_indices], "dense": [float(x) for x in f.core.reshape(-1)]},
        "diagonal": [{"i": int(i), "d": float(d)} for i, d in zip(f.diag_index, f.diag_value)],
    }


def _write(doc, path):
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=1, sort_keys=True)  # nlohmann::json: sorted keys, dump(1)


def _load_flat(path):
    lib = api.library()
    h = api.load_factorization_handle(path)
    try:
        return lib.read_result(h), h
    except Exception:
        lib.result_free(h)
        raise


@pytest.mark.parametrize("name", ["rmat10_m8", "grid32_m16", "rbf256_k3", "rbf512_k4", "zero_cols_bypass",
                                  "partitioned_input", "diag64", "trivial8", "undersize_repair"])
def test_reference_schema_round_trip(name, tmp_path):
    inp, params, part = cases.build(name)
    f = oracles.factorize("oracle", inp, params, part)
    doc = reference_json(f, params)
    src = str(tmp_path / "ref.json")
    _write(doc, src)
    g, h = _load_flat(src)
    lib = api.library()
    try:
        oracles.assert_same(g, f)
        assert g.residual_sq == f.residual_sq
        out = str(tmp_path / "ours.json")
        api.save_factorization(h, out)
    finally:
        lib.result_free(h)
    with open(out) as fh:
        ours = json.load(fh)
    assert ours == doc  # the same document, every double exact
    loaded = api.load_factorization(out)
    assert loaded.params.k == params.k and loaded.params.cluster.m_target == params.m_target
    assert loaded.params.seed == params.seed and loaded.params.eta == params.eta


def test_golden_fixture_round_trip(tmp_path):
    """Reference-generated golden factorizations survive the JSON container
    exactly (checked against the fixture, not just against the writer)."""
    import golden_io

    names = golden_io.names()
    assert names
    for nm in names[:5]:
        inp, params, part, d = golden_io.load(nm)
        f = oracles.factorize("oracle", inp, params, part)
        src = str(tmp_path / f"{nm}.json")
        _write(reference_json(f, params), src)
        g, h = _load_flat(src)
        api.library().result_free(h)
        golden_io.check(g, d)


def test_bad_files(tmp_path):
    inp, params, part = cases.build("rmat10_m8")
    doc = reference_json(oracles.factorize("oracle", inp, params, part), params)
    bad = str(tmp_path / "bad.json")
    for mutate, what in [
        (lambda d: d.update(format="other"), "unknown format"),
        (lambda d: d.update(version=2), "unsupported version"),
        (lambda d: d["core"]["dense"].pop(), "core size mismatch"),
        (lambda d: d["stages"][0]["rotations"][0]["q"].pop(), "rotation matrix size mismatch"),
        (lambda d: d.pop("n"), "missing key"),
        (lambda d: d["params"].update(k=0), "params.k outside"),
        (lambda d: d["params"].update(k=9), "params.k outside"),
        (lambda d: d.update(n=-1), "negative n"),
        (lambda d: d["stages"][0]["rotations"][0]["i"].__setitem__(0, 10 ** 9), "rotation index out of range"),
        (lambda d: d["stages"][0]["rotations"][0]["i"].__setitem__(1, -3), "rotation index out of range"),
        (lambda d: d["stages"][0]["partition"][0].__setitem__(0, 1 << 40), "partition member out of range"),
        (lambda d: d["stages"][0]["eliminated"][0].update(i=-1), "eliminated index out of range"),
        (lambda d: d["core"]["indices"].__setitem__(0, 1 << 30), "core index out of range"),
        (lambda d: d["diagonal"][0].update(i=1 << 30), "diagonal index out of range"),
    ]:
        d = json.loads(json.dumps(doc))
        mutate(d)
        _write(d, bad)
        with pytest.raises(abi.DataError, match=what):
            api.load_factorization(bad)
    with open(bad, "w") as fh:
        fh.write('{"format": "pmmf-factorization", "version": 1,')
    with pytest.raises(abi.DataError):
        api.load_factorization(bad)
    with pytest.raises(abi.DataError, match="cannot open"):
        api.load_factorization(str(tmp_path / "missing.json"))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["rmat12_m16", "grid64_m16", "rbf512_k4"])
def test_gpu_save_load_operator(name, tmp_path):
    """MmfOperator from a reloaded GPU factorization = from the original."""
    lib = api.library()
    inp, params, part = cases.build(name)
    _, h = oracles.result_handle("gpu", inp, params, part)
    path = str(tmp_path / "f.json")
    vecs = np.random.default_rng(3).standard_normal((4, inp[0]))
    outs = []
    try:
        orig = lib.read_result(h)
        api.save_factorization(h, path)
        h2 = api.load_factorization_handle(path)
        oracles.assert_same(lib.read_result(h2), orig)
        for handle in (h, h2):
            op = ctypes.c_void_p()
            err = lib.errbuf()
            abi.raise_for(lib.operator_create(handle, 1e-12, ctypes.byref(op), err, len(err)), err)
            out = np.zeros_like(vecs)
            abi.raise_for(lib.operator_apply(op, 2, 4, vecs.ctypes.data, out.ctypes.data, 0, err, len(err)), err)
            lib.operator_free(op)
            outs.append(out)
        lib.result_free(h2)
    finally:
        lib.result_free(h)
    assert np.array_equal(outs[0], outs[1])
    assert os.path.getsize(path) > 0
