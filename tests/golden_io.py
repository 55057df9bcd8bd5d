"""Reads the golden fixtures written by tests/golden/make_golden.py."""
import glob
import os

import numpy as np

from paper_1507_04396_b200.abi import make_params

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
PFIELDS = ["k", "n_stages", "eta", "m_target", "c_min", "c_max", "d_max", "bypass_enabled", "core_min", "core_cap", "seed"]


def names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")) if not p.endswith("kat.npz"))


def load(name):
    d = np.load(os.path.join(GOLDEN, name + ".npz"))
    pv = d["params"]
    kw = {k: (float(v) if k == "eta" else int(v)) for k, v in zip(PFIELDS, pv)}
    kw["bypass_enabled"] = bool(kw["bypass_enabled"])
    params = make_params(**kw)
    part = None
    if "part_offsets" in d:
        o, m = d["part_offsets"], d["part_members"]
        part = [m[o[i]:o[i + 1]] for i in range(len(o) - 1)]
    inp = (int(d["n"]), d["rows"], d["cols"], d["vals"])
    return inp, params, part, d


def check(f, d):
    """Asserts a FlatFactorization equals the golden record bit-for-bit."""
    assert len(f.stages) == int(d["n_stages_run"])
    assert np.array_equal(f.active_history, d["active_history"])
    for s, st in enumerate(f.stages):
        for fld in ["cluster_offsets", "members", "rot_indices", "rot_matrices", "elim_index", "elim_diagonal",
                    "elim_off_mass_sq", "bypassed"]:
            a, b = getattr(st, fld), d[f"s{s}_{fld}"]
            assert a.shape == b.shape and np.array_equal(a, b), f"stage {s + 1} {fld}"
    assert np.array_equal(f.core_indices, d["core_indices"])
    assert np.array_equal(f.core, d["core"])
    assert np.array_equal(f.diag_index, d["diag_index"]) and np.array_equal(f.diag_value, d["diag_value"])
    assert f.residual_sq == float(d["residual_sq"])
