"""Generates the golden fixtures from the REFERENCE compiled in place
(oracle/_ref/libpmmf_ref.so, built by oracle/Makefile from /root/reference).

Run in the build container (needs /root/reference):  python tests/golden/make_golden.py
Each fixture stores the input triplets (+ partition), the parameters, and
the reference's MmfFactorization in flat arrays, plus an inv_sqrt apply of
three seeded vectors.  Known-answer tests from SPEC.md examples are stored
in kat.npz.
"""
import ctypes
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import cases  # noqa: E402
import oracles  # noqa: E402
from paper_1507_04396_b200 import abi  # noqa: E402

NAMES = ["rmat10_m8", "grid32_m16", "dense256_m2", "rbf256_k3", "zero_cols_bypass", "zero_cols_nobypass",
         "partitioned_input", "dups_and_zeros", "diag64", "trivial8", "undersize_repair", "oversize_recursion",
         "k3_sparse"]
PFIELDS = ["k", "n_stages", "eta", "m_target", "c_min", "c_max", "d_max", "bypass_enabled", "core_min", "core_cap", "seed"]


def dump(name):
    inp, params, part = cases.build(name)
    f = oracles.factorize("ref", inp, params, part)
    vecs = np.random.default_rng(1234).standard_normal((3, inp[0]))
    applied, neg = oracles.operator_apply("ref", inp, params, 2, vecs, clusters=part)
    d = {"n": inp[0], "rows": inp[1], "cols": inp[2], "vals": inp[3],
         "params": np.array([float(getattr(params, k)) for k in PFIELDS]),
         "residual_sq": f.residual_sq, "active_history": f.active_history, "core_indices": f.core_indices,
         "core": f.core, "diag_index": f.diag_index, "diag_value": f.diag_value, "n_stages_run": len(f.stages),
         "apply_in": vecs, "apply_inv_sqrt": applied, "zeroed_negatives": neg}
    if part is not None:
        d["part_offsets"] = np.cumsum([0] + [len(c) for c in part])
        d["part_members"] = np.concatenate(part)
    for s, st in enumerate(f.stages):
        for fld in ["cluster_offsets", "members", "rot_indices", "rot_matrices", "elim_index", "elim_diagonal",
                    "elim_off_mass_sq", "bypassed"]:
            d[f"s{s}_{fld}"] = getattr(st, fld)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
    print(name, len(f.stages), "stages", sum(len(s.rot_indices) for s in f.stages), "rotations")


def kats():
    ref = oracles.load("ref")
    out = {}
    err = ref.errbuf()
    for key, k, g in [("gram_2112", 2, [[2.0, 1.0], [1.0, 2.0]]), ("diag", 2, [[3.0, 0.0], [0.0, 1.0]]),
                      ("k3", 3, [[4.0, 1.0, 0.5], [1.0, 3.0, 0.25], [0.5, 0.25, 2.0]])]:
        g = np.array(g)
        q = np.zeros((k, k))
        abi.raise_for(ref.rotation_from_gram(k, g.ctypes.data_as(abi.c_f64p), q.ctypes.data_as(abi.c_f64p), err, 4096), err)
        out[key + "_g"] = g
        out[key + "_q"] = q
    np.savez_compressed(os.path.join(HERE, "kat.npz"), **out)


if __name__ == "__main__":
    for nm in NAMES:
        dump(nm)
    kats()
