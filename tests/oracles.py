"""Test-only access to the two CPU checkers (never imported by the product):
  * oracle/liboracle.so          — CPU restatement (prefix pmmf_oracle_)
  * oracle/_ref/libpmmf_ref.so   — the reference compiled in place (prefix pmmf_ref_)
"""
import ctypes
import os

import numpy as np

from paper_1507_04396_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE = os.path.join(ROOT, "oracle", "liboracle.so")
REF = os.path.join(ROOT, "oracle", "_ref", "libpmmf_ref.so")

_cache = {}


def load(which: str) -> abi.FlatAbi:
    if which not in _cache:
        if which == "oracle":
            _cache[which] = abi.FlatAbi(ORACLE, "pmmf_oracle_")
        elif which == "ref":
            a = abi.FlatAbi(REF, "pmmf_ref_")
            a.lib.pmmf_ref_set_threads.argtypes = [ctypes.c_int32]
            a.lib.pmmf_ref_residual_frobenius.argtypes = [
                ctypes.c_void_p, ctypes.POINTER(abi.Coo), abi.c_f64p, abi.c_f64p, ctypes.c_char_p, ctypes.c_size_t]
            _cache[which] = a
        elif which == "gpu":
            from paper_1507_04396_b200 import api
            _cache[which] = api.library()
        else:
            raise KeyError(which)
    return _cache[which]


def ref_workload(kind: str, *args):
    """Seeded SURVEY.md §8(d) inputs generated on the reference's own pmmf::Rng
    (oracle/ref_driver.cpp), without loading libpmmf_b200.so.
    kind: rmat(scale, epv, seed, shift) | dense_spd(n, d, seed, shift) |
          rbf(n, dim, bw, seed, shift) | aniso_grid(side, ax, ay)."""
    lib = load("ref").lib
    fn = getattr(lib, "pmmf_ref_workload_" + kind)
    sig = {"rmat": [ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double],
           "dense_spd": [ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double],
           "rbf": [ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_uint64, ctypes.c_double],
           "aniso_grid": [ctypes.c_int64, ctypes.c_double, ctypes.c_double]}[kind]
    fn.argtypes = sig + [ctypes.POINTER(abi.Workload)]
    fn.restype = ctypes.c_int
    lib.pmmf_ref_workload_free.argtypes = [ctypes.POINTER(abi.Workload)]
    w = abi.Workload()
    if fn(*args, ctypes.byref(w)):
        raise ValueError(f"ref workload {kind}{args}: bad arguments")
    try:
        m = w.nnz
        rows = np.ctypeslib.as_array(w.rows, (m,)).copy() if m else np.zeros(0, np.int64)
        cols = np.ctypeslib.as_array(w.cols, (m,)).copy() if m else np.zeros(0, np.int64)
        vals = np.ctypeslib.as_array(w.vals, (m,)).copy() if m else np.zeros(0)
        return int(w.n), rows, cols, vals
    finally:
        lib.pmmf_ref_workload_free(ctypes.byref(w))


def available(which: str) -> bool:
    return os.path.exists({"oracle": ORACLE, "ref": REF}[which])


def factorize(which, inp, params, clusters=None, comm=None):
    """Runs one factorization through a flat ABI; returns FlatFactorization.
    comm (gpu only): an api.Communicator for the sharded entry point."""
    lib = load(which)
    n, rows, cols, vals = inp
    coo, keep = abi.make_coo(n, rows, cols, vals, clusters)
    h = ctypes.c_void_p()
    err = lib.errbuf()
    if comm is None:
        st = lib.factorize(ctypes.byref(coo), ctypes.byref(params), ctypes.byref(h), err, len(err))
    else:
        st = lib.lib.pmmf_b200_factorize_sharded(ctypes.byref(coo), ctypes.byref(params), comm.handle,
                                                 ctypes.byref(h), err, len(err))
    abi.raise_for(st, err)
    try:
        return lib.read_result(h)
    finally:
        lib.result_free(h)


def assert_same(a, b, check_mass=True):
    """Bit-for-bit comparison of two flat factorizations; raises with the first difference."""
    assert a.n == b.n and a.k == b.k
    assert np.array_equal(a.active_history, b.active_history), (a.active_history, b.active_history)
    assert len(a.stages) == len(b.stages)
    for s, (x, y) in enumerate(zip(a.stages, b.stages)):
        for f in ["cluster_offsets", "members", "rot_indices", "rot_matrices", "elim_index", "elim_diagonal", "bypassed"]:
            u, v = getattr(x, f), getattr(y, f)
            if not (u.shape == v.shape and np.array_equal(u, v)):
                raise AssertionError(f"stage {s + 1}: field {f} differs")
        if check_mass and not np.array_equal(x.elim_off_mass_sq, y.elim_off_mass_sq):
            raise AssertionError(f"stage {s + 1}: elim_off_mass_sq differs")
    assert np.array_equal(a.core_indices, b.core_indices)
    assert np.array_equal(a.core, b.core), "core differs"
    assert np.array_equal(a.diag_index, b.diag_index)
    assert np.array_equal(a.diag_value, b.diag_value), "retired diagonal differs"
    if check_mass:
        assert a.residual_sq == b.residual_sq, (a.residual_sq, b.residual_sq)


def result_handle(which, inp, params, clusters=None):
    lib = load(which)
    n, rows, cols, vals = inp
    coo, keep = abi.make_coo(n, rows, cols, vals, clusters)
    h = ctypes.c_void_p()
    err = lib.errbuf()
    abi.raise_for(lib.factorize(ctypes.byref(coo), ctypes.byref(params), ctypes.byref(h), err, len(err)), err)
    return lib, h


def operator_apply(which, inp, params, mode, vecs, thr=1e-12, clusters=None):
    """Factorize, build the MmfOperator, apply `mode` to the rhs-major vecs."""
    lib, h = result_handle(which, inp, params, clusters)
    op = ctypes.c_void_p()
    err = lib.errbuf()
    try:
        abi.raise_for(lib.operator_create(h, thr, ctypes.byref(op), err, len(err)), err)
    finally:
        lib.result_free(h)
    try:
        vecs = np.ascontiguousarray(vecs, np.float64)
        out = np.zeros_like(vecs)
        nrhs = vecs.shape[0]
        abi.raise_for(lib.operator_apply(op, mode, nrhs, vecs.ctypes.data, out.ctypes.data, 0, err, len(err)), err)
        neg = ctypes.c_int64()
        lib.operator_zeroed_negatives(op, ctypes.byref(neg))
        return out, neg.value
    finally:
        lib.operator_free(op)


def solve(which, inp, params, tol, max_iter, rhs_count, seed, precondition=True):
    """run_solve_experiment through a flat ABI: returns (iters, conv, brk, traces, wall_ms)."""
    lib, h = result_handle(which, inp, params) if precondition else (load(which), None)
    op = ctypes.c_void_p()
    err = lib.errbuf()
    if precondition:
        try:
            abi.raise_for(lib.operator_create(h, 1e-12, ctypes.byref(op), err, len(err)), err)
        finally:
            lib.result_free(h)
    n, rows, cols, vals = inp
    coo, keep = abi.make_coo(n, rows, cols, vals)
    cfg = abi.SolveConfig(tol, max_iter, rhs_count, seed)
    it = np.zeros(rhs_count, np.int32)
    cv = np.zeros(rhs_count, np.int32)
    bk = np.zeros(rhs_count, np.int32)
    tr = np.zeros((rhs_count, max_iter + 1))
    wall = ctypes.c_double()
    try:
        abi.raise_for(
            lib.solve(ctypes.byref(coo), op if precondition else None, ctypes.byref(cfg),
                      it.ctypes.data_as(abi.c_i32p), cv.ctypes.data_as(abi.c_i32p), bk.ctypes.data_as(abi.c_i32p),
                      tr.ctypes.data_as(abi.c_f64p), ctypes.byref(wall), err, len(err)), err)
    finally:
        if precondition:
            lib.operator_free(op)
    return it, cv, bk, tr, wall.value


# ---- comparison preconditioners and Nystrom (solver.hpp:222-349, transform_ops.hpp:252-307)
PRECOND = {"none": 0, "jacobi": 1, "ssor": 2, "ic": 3, "pmmf": 4}


def precond_apply(which, inp, kind, vecs, side, omega=1.0, part=None):
    """K^-1 (side 0) or K^-T (side 1) of a comparison preconditioner on the
    rows of `vecs`; returns (out, (kind, compensated, alpha))."""
    lib = load(which)
    n, rows, cols, vals = inp
    coo, keep = abi.make_coo(n, rows, cols, vals, clusters=part)
    err = lib.errbuf()
    pc = ctypes.c_void_p()
    abi.raise_for(lib.precond_create(ctypes.byref(coo), PRECOND[kind], omega, ctypes.byref(pc), err, len(err)), err)
    try:
        vecs = np.ascontiguousarray(vecs, dtype=np.float64)
        out = np.zeros_like(vecs)
        abi.raise_for(lib.precond_apply(pc, side, vecs.shape[0], vecs.ctypes.data, out.ctypes.data, 0, err, len(err)),
                      err)
        k, c, a = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_double()
        lib.precond_info(pc, ctypes.byref(k), ctypes.byref(c), ctypes.byref(a))
        return out, (k.value, c.value, a.value)
    finally:
        lib.precond_free(pc)


def solve_precond(which, inp, kind, tol, max_iter, rhs_count, seed, omega=1.0):
    """run_solve_experiment with a comparison preconditioner (kind "none" =
    plain CG): returns (iters, conv, brk, traces, wall_ms)."""
    lib = load(which)
    n, rows, cols, vals = inp
    coo, keep = abi.make_coo(n, rows, cols, vals)
    err = lib.errbuf()
    pc = ctypes.c_void_p()
    if kind != "none":
        abi.raise_for(lib.precond_create(ctypes.byref(coo), PRECOND[kind], omega, ctypes.byref(pc), err, len(err)),
                      err)
    cfg = abi.SolveConfig(tol, max_iter, rhs_count, seed)
    it = np.zeros(rhs_count, np.int32)
    cv = np.zeros(rhs_count, np.int32)
    bk = np.zeros(rhs_count, np.int32)
    tr = np.zeros((rhs_count, max_iter + 1))
    wall = ctypes.c_double()
    try:
        abi.raise_for(
            lib.solve_precond(ctypes.byref(coo), pc if kind != "none" else None, ctypes.byref(cfg),
                              it.ctypes.data_as(abi.c_i32p), cv.ctypes.data_as(abi.c_i32p),
                              bk.ctypes.data_as(abi.c_i32p), tr.ctypes.data_as(abi.c_f64p), ctypes.byref(wall), err,
                              len(err)), err)
    finally:
        if kind != "none":
            lib.precond_free(pc)
    return it, cv, bk, tr, wall.value


def nystrom(which, inp, m, seed, cap=4096, part=None):
    """nystrom_uniform: returns (frobenius_error, columns)."""
    lib = load(which)
    n, rows, cols, vals = inp
    coo, keep = abi.make_coo(n, rows, cols, vals, clusters=part)
    err = lib.errbuf()
    fro = ctypes.c_double()
    sel = np.zeros(max(int(m), 1), np.int64)
    abi.raise_for(lib.nystrom_uniform(ctypes.byref(coo), m, seed, cap, ctypes.byref(fro),
                                      sel.ctypes.data_as(abi.c_i64p), err, len(err)), err)
    return fro.value, sel[:m]
