"""ctypes mirror of include/pmmf_b200.h and include/pmmf_b200_workloads.h.

The same flat C-ABI shape is exported by three libraries:
  * ``libpmmf_b200.so``           — the product (prefix ``pmmf_b200_``),
  * ``oracle/liboracle.so``       — the CPU restatement (prefix ``pmmf_oracle_``),
  * ``oracle/_ref/libpmmf_ref.so``— the reference compiled in place (prefix ``pmmf_ref_``).
``FlatAbi`` binds one of them by prefix; only tests / bench may bind the oracles.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

c_i64p = ctypes.POINTER(ctypes.c_int64)
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_f64p = ctypes.POINTER(ctypes.c_double)

STATUS_NAMES = {
    0: "OK",
    1: "INVALID_ARGUMENT",
    2: "OUT_OF_RANGE",
    3: "NUMERIC",
    4: "DATA",
    5: "CUDA",
    6: "INTERNAL",
}


class PmmfError(RuntimeError):
    """Base of the status-code exceptions (types.hpp:24-32 error convention)."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class InvalidArgument(PmmfError, ValueError):
    pass


class OutOfRange(PmmfError, IndexError):
    pass


class NumericError(PmmfError, ArithmeticError):
    pass


class DataError(PmmfError):
    pass


class CudaError(PmmfError):
    pass


_EXC = {1: InvalidArgument, 2: OutOfRange, 3: NumericError, 4: DataError, 5: CudaError}


def raise_for(status: int, err: ctypes.Array) -> None:
    if status == 0:
        return
    msg = err.value.decode(errors="replace") if err is not None else ""
    raise _EXC.get(status, PmmfError)(status, f"[{STATUS_NAMES.get(status, status)}] {msg}")


class Params(ctypes.Structure):
    _fields_ = [
        ("k", ctypes.c_int32),
        ("n_stages", ctypes.c_int32),
        ("eta", ctypes.c_double),
        ("m_target", ctypes.c_int64),
        ("c_min", ctypes.c_int64),
        ("c_max", ctypes.c_int64),
        ("d_max", ctypes.c_int32),
        ("bypass_enabled", ctypes.c_int32),
        ("cluster_seed", ctypes.c_uint64),
        ("core_min", ctypes.c_int64),
        ("core_cap", ctypes.c_int64),
        ("seed", ctypes.c_uint64),
    ]


class Coo(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("nnz", ctypes.c_int64),
        ("rows", ctypes.c_void_p),
        ("cols", ctypes.c_void_p),
        ("vals", ctypes.c_void_p),
        ("n_clusters", ctypes.c_int64),
        ("cluster_offsets", ctypes.c_void_p),
        ("cluster_members", ctypes.c_void_p),
        ("on_device", ctypes.c_int32),
        ("device", ctypes.c_int32),
    ]


class Summary(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("n_stages", ctypes.c_int64),
        ("k", ctypes.c_int64),
        ("core_size", ctypes.c_int64),
        ("n_diagonal", ctypes.c_int64),
        ("trivial", ctypes.c_int64),
        ("residual_sq", ctypes.c_double),
    ]


class StageSizes(ctypes.Structure):
    _fields_ = [
        ("n_clusters", ctypes.c_int64),
        ("partition_size", ctypes.c_int64),
        ("n_rotations", ctypes.c_int64),
        ("n_eliminated", ctypes.c_int64),
        ("n_bypassed", ctypes.c_int64),
    ]


class SolveConfig(ctypes.Structure):
    _fields_ = [
        ("tol", ctypes.c_double),
        ("max_iter", ctypes.c_int32),
        ("rhs_count", ctypes.c_int32),
        ("seed", ctypes.c_uint64),
    ]


class Workload(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("nnz", ctypes.c_int64),
        ("rows", c_i64p),
        ("cols", c_i64p),
        ("vals", c_f64p),
    ]


def ptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    return ctypes.c_void_p(a.ctypes.data)


# ---------------------------------------------------------------- results
@dataclass
class FlatStage:
    """One ``Stage`` (factorizer.hpp:65-70) in flat arrays."""

    cluster_offsets: np.ndarray
    members: np.ndarray
    rot_indices: np.ndarray  # (R, k)
    rot_matrices: np.ndarray  # (R, k, k)
    elim_index: np.ndarray
    elim_diagonal: np.ndarray
    elim_off_mass_sq: np.ndarray
    bypassed: np.ndarray

    def clusters(self) -> List[np.ndarray]:
        o = self.cluster_offsets
        return [self.members[o[u] : o[u + 1]] for u in range(len(o) - 1)]


@dataclass
class FlatFactorization:
    """``MmfFactorization`` (factorizer.hpp:111-118) + ``FactorizeStats``."""

    n: int
    k: int
    residual_sq: float
    trivial: bool
    active_history: np.ndarray
    stages: List[FlatStage]
    core_indices: np.ndarray
    core: np.ndarray
    diag_index: np.ndarray
    diag_value: np.ndarray
    phases: np.ndarray = field(default_factory=lambda: np.zeros(6))
    stage_info: np.ndarray = field(default_factory=lambda: np.zeros((0, 7), np.int64))


class FlatAbi:
    """Binds the flat C-ABI of one library under a symbol prefix."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"library not built: {path}")
        self.path = path
        self.prefix = prefix
        self.lib = ctypes.CDLL(path)
        L = self.lib

        def fn(name, restype, argtypes):
            f = getattr(L, prefix + name)
            f.restype = restype
            f.argtypes = argtypes
            return f

        E = [ctypes.c_char_p, ctypes.c_size_t]
        V = ctypes.c_void_p
        self.factorize = fn("factorize", ctypes.c_int, [ctypes.POINTER(Coo), ctypes.POINTER(Params), ctypes.POINTER(V)] + E)
        self.result_summary = fn("result_summary", ctypes.c_int, [V, ctypes.POINTER(Summary)])
        self.result_active_history = fn("result_active_history", ctypes.c_int, [V, c_i64p])
        self.result_stage_sizes = fn("result_stage_sizes", ctypes.c_int, [V, ctypes.c_int64, ctypes.POINTER(StageSizes)])
        self.result_stage = fn(
            "result_stage",
            ctypes.c_int,
            [V, ctypes.c_int64, c_i64p, c_i64p, c_i64p, c_f64p, c_i64p, c_f64p, c_f64p, c_i64p],
        )
        self.result_core = fn("result_core", ctypes.c_int, [V, c_i64p, c_f64p, c_i64p, c_f64p])
        self.result_stats = fn("result_stats", ctypes.c_int, [V, c_f64p, c_i64p])
        self.result_free = fn("result_free", None, [V])
        self.operator_create = fn("operator_create", ctypes.c_int, [V, ctypes.c_double, ctypes.POINTER(V)] + E)
        self.operator_apply = fn(
            "operator_apply", ctypes.c_int, [V, ctypes.c_int32, ctypes.c_int64, V, V, ctypes.c_int32] + E
        )
        self.operator_zeroed_negatives = fn("operator_zeroed_negatives", ctypes.c_int, [V, c_i64p])
        self.operator_free = fn("operator_free", None, [V])
        self.solve = fn(
            "solve",
            ctypes.c_int,
            [ctypes.POINTER(Coo), V, ctypes.POINTER(SolveConfig), c_i32p, c_i32p, c_i32p, c_f64p, c_f64p] + E,
        )
        self.rotation_from_gram = fn("rotation_from_gram", ctypes.c_int, [ctypes.c_int32, c_f64p, c_f64p] + E)
        # comparison preconditioners + Nystrom (solver.hpp:222-349, transform_ops.hpp:252-307)
        self.precond_create = fn("precond_create", ctypes.c_int,
                                 [ctypes.POINTER(Coo), ctypes.c_int32, ctypes.c_double, ctypes.POINTER(V)] + E)
        self.precond_from_operator = fn("precond_from_operator", ctypes.c_int, [V, ctypes.POINTER(V)] + E)
        self.precond_apply = fn("precond_apply", ctypes.c_int,
                                [V, ctypes.c_int32, ctypes.c_int64, V, V, ctypes.c_int32] + E)
        self.precond_info = fn("precond_info", ctypes.c_int, [V, c_i32p, c_i32p, c_f64p])
        self.precond_free = fn("precond_free", None, [V])
        self.solve_precond = fn(
            "solve_precond",
            ctypes.c_int,
            [ctypes.POINTER(Coo), V, ctypes.POINTER(SolveConfig), c_i32p, c_i32p, c_i32p, c_f64p, c_f64p] + E,
        )
        self.nystrom_uniform = fn("nystrom_uniform", ctypes.c_int,
                                  [ctypes.POINTER(Coo), ctypes.c_int64, ctypes.c_uint64, ctypes.c_int64, c_f64p,
                                   c_i64p] + E)

    # ------------------------------------------------------------------
    @staticmethod
    def errbuf():
        return ctypes.create_string_buffer(4096)

    def read_result(self, h) -> FlatFactorization:
        s = Summary()
        raise_for(self.result_summary(h, ctypes.byref(s)), None)
        ns = s.n_stages
        hist = np.zeros(ns + 1, np.int64)
        self.result_active_history(h, hist.ctypes.data_as(c_i64p))
        stages = []
        for st in range(ns):
            sz = StageSizes()
            raise_for(self.result_stage_sizes(h, st, ctypes.byref(sz)), None)
            k = s.k
            off = np.zeros(sz.n_clusters + 1, np.int64)
            mem = np.zeros(max(sz.partition_size, 1), np.int64)
            ri = np.zeros((max(sz.n_rotations, 1), k), np.int64)
            rq = np.zeros((max(sz.n_rotations, 1), k, k), np.float64)
            ei = np.zeros(max(sz.n_eliminated, 1), np.int64)
            ed = np.zeros(max(sz.n_eliminated, 1), np.float64)
            em = np.zeros(max(sz.n_eliminated, 1), np.float64)
            by = np.zeros(max(sz.n_bypassed, 1), np.int64)
            raise_for(
                self.result_stage(
                    h,
                    st,
                    off.ctypes.data_as(c_i64p),
                    mem.ctypes.data_as(c_i64p),
                    ri.ctypes.data_as(c_i64p),
                    rq.ctypes.data_as(c_f64p),
                    ei.ctypes.data_as(c_i64p),
                    ed.ctypes.data_as(c_f64p),
                    em.ctypes.data_as(c_f64p),
                    by.ctypes.data_as(c_i64p),
                ),
                None,
            )
            stages.append(
                FlatStage(
                    off,
                    mem[: sz.partition_size],
                    ri[: sz.n_rotations],
                    rq[: sz.n_rotations],
                    ei[: sz.n_eliminated],
                    ed[: sz.n_eliminated],
                    em[: sz.n_eliminated],
                    by[: sz.n_bypassed],
                )
            )
        g = s.core_size
        ci = np.zeros(max(g, 1), np.int64)
        core = np.zeros((max(g, 1), max(g, 1)), np.float64)
        di = np.zeros(max(s.n_diagonal, 1), np.int64)
        dv = np.zeros(max(s.n_diagonal, 1), np.float64)
        raise_for(
            self.result_core(h, ci.ctypes.data_as(c_i64p), core.ctypes.data_as(c_f64p), di.ctypes.data_as(c_i64p), dv.ctypes.data_as(c_f64p)),
            None,
        )
        core = core.reshape(-1)[: g * g].reshape(g, g) if g else np.zeros((0, 0))
        phases = np.zeros(6)
        info = np.zeros((max(ns, 1), 7), np.int64)
        self.result_stats(h, phases.ctypes.data_as(c_f64p), info.ctypes.data_as(c_i64p))
        return FlatFactorization(
            n=s.n,
            k=s.k,
            residual_sq=s.residual_sq,
            trivial=bool(s.trivial),
            active_history=hist,
            stages=stages,
            core_indices=ci[:g],
            core=core,
            diag_index=di[: s.n_diagonal],
            diag_value=dv[: s.n_diagonal],
            phases=phases,
            stage_info=info[:ns],
        )


def _check_device_triplets(rows, cols, vals, device):
    """Device triplets must be CUDA tensors on `device`, contiguous, int64 /
    int64 / float64 and of equal length (the C-ABI reads them as raw
    pointers, include/pmmf_b200.h)."""
    import torch

    want = (torch.int64, torch.int64, torch.float64)
    for name, x, dt in zip(("rows", "cols", "vals"), (rows, cols, vals), want):
        if not getattr(x, "is_cuda", False):
            raise ValueError(f"device input: {name} is not a CUDA tensor")
        if x.dtype != dt:
            raise ValueError(f"device input: {name} has dtype {x.dtype}, expected {dt}")
        if not x.is_contiguous():
            raise ValueError(f"device input: {name} is not contiguous")
        if x.device.index != int(device):
            raise ValueError(f"device input: {name} lives on cuda:{x.device.index}, the call targets cuda:{device}")
    if not (rows.numel() == cols.numel() == vals.numel()):
        raise ValueError(f"device input: lengths differ ({rows.numel()}, {cols.numel()}, {vals.numel()})")


def make_coo(n, rows, cols, vals, clusters=None, on_device=False, device=0, keep=None):
    """Builds a Coo struct; ``keep`` collects the arrays that must outlive it."""
    keep = [] if keep is None else keep
    c = Coo()
    c.n = int(n)
    if on_device:
        _check_device_triplets(rows, cols, vals, device)
        c.nnz = int(rows.numel())
        c.rows, c.cols, c.vals = rows.data_ptr(), cols.data_ptr(), vals.data_ptr()
        keep += [rows, cols, vals]
    else:
        if hasattr(rows, "is_cuda"):  # CPU torch tensors: host buffers
            rows, cols, vals = (x.numpy() for x in (rows, cols, vals))
        rows = np.ascontiguousarray(rows, np.int64)
        cols = np.ascontiguousarray(cols, np.int64)
        vals = np.ascontiguousarray(vals, np.float64)
        keep += [rows, cols, vals]
        c.nnz = int(rows.size)
        c.rows, c.cols, c.vals = rows.ctypes.data, cols.ctypes.data, vals.ctypes.data
    if clusters is None:
        c.n_clusters = 0
    else:
        offs = np.zeros(len(clusters) + 1, np.int64)
        offs[1:] = np.cumsum([len(x) for x in clusters])
        mem = np.concatenate([np.asarray(x, np.int64) for x in clusters]) if clusters else np.zeros(0, np.int64)
        mem = np.ascontiguousarray(mem, np.int64)
        keep += [offs, mem]
        c.n_clusters = len(clusters)
        c.cluster_offsets = offs.ctypes.data
        c.cluster_members = mem.ctypes.data
    c.on_device = 1 if on_device else 0
    c.device = int(device)
    return c, keep


def make_params(k=2, n_stages=15, eta=0.5, m_target=2, c_min=10, c_max=5000, d_max=500, bypass_enabled=True, core_min=10, core_cap=4096, seed=0, cluster_seed=0) -> Params:
    """Defaults follow FactorizeParams / ClusterParams (factorizer.hpp:35-51, clustering.hpp:28-41)."""
    p = Params()
    p.k, p.n_stages, p.eta = k, n_stages, eta
    p.m_target, p.c_min, p.c_max, p.d_max = m_target, c_min, c_max, d_max
    p.bypass_enabled = 1 if bypass_enabled else 0
    p.cluster_seed = cluster_seed
    p.core_min, p.core_cap, p.seed = core_min, core_cap, seed
    return p


# ------------------------------------------------------------- input path
class Triplets(ctypes.Structure):
    """pmmf_b200_triplets: TripletMatrix / EdgeList (io.hpp:27-33, :150-154)."""

    _fields_ = [("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("row", c_i64p), ("col", c_i64p), ("val", c_f64p), ("n_ids", ctypes.c_int64),
                ("original_ids", c_i64p)]


class IoAbi:
    """The io.hpp entry points of one library (pmmf_b200_ or the reference's pmmf_ref_)."""

    def __init__(self, lib: ctypes.CDLL, prefix: str, device_args: bool):
        E = [ctypes.c_char_p, ctypes.c_size_t]
        V = ctypes.c_void_p
        self.prefix, self.device_args = prefix, device_args

        def fn(name, argtypes):
            f = getattr(lib, prefix + name)
            f.restype = ctypes.c_int
            f.argtypes = argtypes
            return f

        TP = ctypes.POINTER(ctypes.POINTER(Triplets))
        self.read_mm = fn("read_matrix_market", [ctypes.c_char_p, TP] + E)
        self.read_el = fn("read_edge_list", [ctypes.c_char_p, TP] + E)
        self.free = getattr(lib, prefix + "triplets_free")
        self.free.restype = None
        self.free.argtypes = [ctypes.POINTER(Triplets)]
        self.write_mm = fn("write_matrix_market", [ctypes.c_char_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                                    V, V, V] + E)
        dev = [ctypes.c_int32, ctypes.c_int32] if device_args else []
        self.lap = fn("laplacian", [ctypes.c_int64, ctypes.c_int64, V, V, V, ctypes.c_double] + dev + [V, V, V] + E)
        self.sym = fn("symmetrize", [ctypes.c_int64, V, V, V] + dev + [ctypes.POINTER(ctypes.c_int64), V, V, V] + E)

    @staticmethod
    def _take(t):
        c = t.contents
        n = c.nnz
        r = np.ctypeslib.as_array(c.row, (max(n, 1),))[:n].copy()
        cc = np.ctypeslib.as_array(c.col, (max(n, 1),))[:n].copy()
        v = np.ctypeslib.as_array(c.val, (max(n, 1),))[:n].copy()
        ids = None
        if c.original_ids:
            ids = np.ctypeslib.as_array(c.original_ids, (max(c.n_ids, 1),))[:c.n_ids].copy()
        return c.rows, c.cols, r, cc, v, ids

    def read(self, kind: str, path: str):
        t = ctypes.POINTER(Triplets)()
        err = ctypes.create_string_buffer(4096)
        f = self.read_mm if kind == "mm" else self.read_el
        raise_for(f(os.fsencode(path), ctypes.byref(t), err, len(err)), err)
        try:
            return self._take(t)
        finally:
            self.free(t)

    def write_matrix_market(self, path, rows, cols, r, c, v):
        r, c, v = (np.ascontiguousarray(x, t) for x, t in ((r, np.int64), (c, np.int64), (v, np.float64)))
        err = ctypes.create_string_buffer(4096)
        raise_for(self.write_mm(os.fsencode(path), int(rows), int(cols), len(v), ptr(r), ptr(c), ptr(v), err,
                                len(err)), err)

    def laplacian(self, r, c, v, n, shift=0.0, device=0):
        r, c, v = (np.ascontiguousarray(x, t) for x, t in ((r, np.int64), (c, np.int64), (v, np.float64)))
        m = len(v) + int(n)
        o = (np.zeros(m, np.int64), np.zeros(m, np.int64), np.zeros(m, np.float64))
        err = ctypes.create_string_buffer(4096)
        dev = [0, int(device)] if self.device_args else []
        raise_for(self.lap(int(n), len(v), ptr(r), ptr(c), ptr(v), float(shift), *dev, ptr(o[0]), ptr(o[1]),
                           ptr(o[2]), err, len(err)), err)
        return o

    def symmetrize(self, r, c, v, device=0):
        r, c, v = (np.ascontiguousarray(x, t) for x, t in ((r, np.int64), (c, np.int64), (v, np.float64)))
        m = 2 * len(v)
        o = (np.zeros(max(m, 1), np.int64), np.zeros(max(m, 1), np.int64), np.zeros(max(m, 1), np.float64))
        cnt = ctypes.c_int64()
        err = ctypes.create_string_buffer(4096)
        dev = [0, int(device)] if self.device_args else []
        raise_for(self.sym(len(v), ptr(r), ptr(c), ptr(v), *dev, ctypes.byref(cnt), ptr(o[0]), ptr(o[1]), ptr(o[2]),
                           err, len(err)), err)
        k = cnt.value
        return o[0][:k], o[1][:k], o[2][:k]
