"""Python mirror of the reference's public interface for the stage-loop path.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/pmmf:
  * ``ClusterParams`` / ``FactorizeParams``  (clustering.hpp:28-41, factorizer.hpp:35-51)
  * ``Partition``                           (partition.hpp:19-93)
  * ``BlockedSparseMatrix.from_triplets``   (blocked_matrix.hpp:133-156)
  * ``factorize``                           (factorizer.hpp:397-595)
  * ``MmfOperator`` / ``apply*``            (transform_ops.hpp:30-153)
  * ``run_solve_experiment``                (solver.hpp:368-416)
Everything executes in ``libpmmf_b200.so`` (hand-written sm_100a kernels);
there is no CPU fallback: a missing library or device raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import abi

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpmmf_b200.so")

_ABI: Optional[abi.FlatAbi] = None


def library() -> abi.FlatAbi:
    """Loads libpmmf_b200.so (fails loudly when it has not been built)."""
    global _ABI
    if _ABI is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libpmmf_b200.so is not built ({LIB_PATH}); run __graft_entry__.build()")
        _ABI = abi.FlatAbi(LIB_PATH, "pmmf_b200_")
        L = _ABI.lib
        L.pmmf_b200_kernel_launches.restype = ctypes.c_int64
        L.pmmf_b200_version.restype = ctypes.c_char_p
        for name in ("rmat", "dense_spd", "rbf", "aniso_grid"):
            getattr(L, "pmmf_b200_workload_" + name).restype = ctypes.c_int
        L.pmmf_b200_workload_free.argtypes = [ctypes.POINTER(abi.Workload)]
        E = [ctypes.c_char_p, ctypes.c_size_t]
        V = ctypes.c_void_p
        L.pmmf_b200_comm_unique_id.restype = ctypes.c_int
        L.pmmf_b200_comm_unique_id.argtypes = [ctypes.c_char_p] + E
        L.pmmf_b200_comm_create.restype = ctypes.c_int
        L.pmmf_b200_comm_create.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_char_p, ctypes.c_int32,
                                            ctypes.POINTER(V)] + E
        L.pmmf_b200_comm_create_virtual.restype = ctypes.c_int
        L.pmmf_b200_comm_create_virtual.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(V)] + E
        L.pmmf_b200_comm_free.restype = None
        L.pmmf_b200_comm_free.argtypes = [V]
        L.pmmf_b200_factorize_sharded.restype = ctypes.c_int
        L.pmmf_b200_factorize_sharded.argtypes = [ctypes.POINTER(abi.Coo), ctypes.POINTER(abi.Params), V,
                                                  ctypes.POINTER(V)] + E
        L.pmmf_b200_result_save.restype = ctypes.c_int
        L.pmmf_b200_result_save.argtypes = [V, ctypes.c_char_p] + E
        L.pmmf_b200_result_load.restype = ctypes.c_int
        L.pmmf_b200_result_load.argtypes = [ctypes.c_char_p, ctypes.POINTER(V)] + E
        L.pmmf_b200_result_params.restype = ctypes.c_int
        L.pmmf_b200_result_params.argtypes = [V, ctypes.POINTER(abi.Params)]
        L.pmmf_b200_residual_frobenius.restype = ctypes.c_int
        L.pmmf_b200_residual_frobenius.argtypes = [V, ctypes.POINTER(abi.Coo), ctypes.c_int32, ctypes.c_int64,
                                                   ctypes.POINTER(ctypes.c_double)] + E
        L.pmmf_b200_shard_ranges.restype = ctypes.c_int
        L.pmmf_b200_shard_ranges.argtypes = [ctypes.c_int64, V, V, ctypes.c_int32, V]
        L.pmmf_b200_result_create.restype = ctypes.c_int
        L.pmmf_b200_result_create.argtypes = [ctypes.c_int64, ctypes.POINTER(abi.Params), ctypes.c_double,
                                              ctypes.POINTER(V)] + E
        L.pmmf_b200_result_add_stage.restype = ctypes.c_int
        L.pmmf_b200_result_add_stage.argtypes = [V, ctypes.c_int64, V, V, ctypes.c_int64, V, V, ctypes.c_int64, V, V, V,
                                                 ctypes.c_int64, V] + E
        L.pmmf_b200_result_set_core.restype = ctypes.c_int
        L.pmmf_b200_result_set_core.argtypes = [V, ctypes.c_int64, V, V, ctypes.c_int64, V, V, V, ctypes.c_int64] + E
    return _ABI


# ------------------------------------------------------------ multi-GPU
COMM_ID_BYTES = 128


class Communicator:
    """The ranks a sharded factorization runs on: one
    process per GPU over NCCL, or `virtual` ranks run one after another in
    this process on one GPU (parity test hook).  The reference's analogue is
    the fork-join pool over a stage's clusters (parallel.hpp:25-71)."""

    def __init__(self, nranks: int, rank: int = 0, device: int = 0, unique_id: Optional[bytes] = None,
                 virtual: bool = False):
        lib = library()
        self.nranks, self.rank, self.device, self.virtual = int(nranks), int(rank), int(device), bool(virtual)
        self.handle = ctypes.c_void_p()
        err = lib.errbuf()
        if virtual:
            st = lib.lib.pmmf_b200_comm_create_virtual(self.nranks, self.device, ctypes.byref(self.handle), err,
                                                       len(err))
        else:
            if self.nranks > 1 and (unique_id is None or len(unique_id) != COMM_ID_BYTES):
                raise ValueError("Communicator: a 128-byte unique id from rank 0 is required")
            st = lib.lib.pmmf_b200_comm_create(self.nranks, self.rank, unique_id, self.device,
                                               ctypes.byref(self.handle), err, len(err))
        abi.raise_for(st, err)

    @staticmethod
    def unique_id() -> bytes:
        lib = library()
        buf = ctypes.create_string_buffer(COMM_ID_BYTES)
        err = lib.errbuf()
        abi.raise_for(lib.lib.pmmf_b200_comm_unique_id(buf, err, len(err)), err)
        return buf.raw

    @classmethod
    def from_torch_distributed(cls, device: int) -> "Communicator":
        """Collective over an initialised torch.distributed group: rank 0
        makes the NCCL id, the group broadcasts it."""
        import torch.distributed as dist

        rank, world = dist.get_rank(), dist.get_world_size()
        box = [cls.unique_id() if rank == 0 and world > 1 else None]
        if world > 1:
            dist.broadcast_object_list(box, src=0)
        return cls(world, rank, device, box[0])

    def close(self) -> None:
        if self.handle:
            library().lib.pmmf_b200_comm_free(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def shard_ranges(sizes, nnz, nranks: int) -> np.ndarray:
    """The cluster split of a sharded stage: contiguous ranges lo[0..nranks]."""
    sizes = np.ascontiguousarray(sizes, np.int64)
    z = None if nnz is None else np.ascontiguousarray(nnz, np.int64)
    lo = np.zeros(int(nranks) + 1, np.int64)
    st = library().lib.pmmf_b200_shard_ranges(len(sizes), abi.ptr(sizes), abi.ptr(z), int(nranks), abi.ptr(lo))
    abi.raise_for(st, None)
    return lo


def set_dense_gram(mode: int) -> None:
    """Dense-cluster Gram kernel (pmmf_b200_set_dense_gram): 0 = bitwise SIMT
    SYRK (default), 1 = FP64 tensor cores (DMMA; the near-tie clause)."""
    L = library().lib
    L.pmmf_b200_set_dense_gram.argtypes = [ctypes.c_int32]
    L.pmmf_b200_set_dense_gram.restype = ctypes.c_int
    if L.pmmf_b200_set_dense_gram(int(mode)) != 0:
        raise abi.InvalidArgument(1, "set_dense_gram: mode must be 0 or 1")


def get_dense_gram() -> int:
    L = library().lib
    L.pmmf_b200_get_dense_gram.restype = ctypes.c_int32
    return int(L.pmmf_b200_get_dense_gram())


def kernel_launches() -> int:
    return int(library().lib.pmmf_b200_kernel_launches())


def cached_device_bytes(device: int = 0, release: bool = False) -> int:
    """Bytes of large device blocks the library keeps for reuse between
    factorizations; release=True hands them back to the device."""
    f = library().lib.pmmf_b200_cached_bytes
    f.restype = ctypes.c_int64
    f.argtypes = [ctypes.c_int32, ctypes.c_int32]
    return int(f(int(device), 1 if release else 0))


# ------------------------------------------------------------------ params
@dataclass
class ClusterParams:
    m_target: int = 2
    c_min: int = 10
    c_max: int = 5000
    d_max: int = 500
    bypass_enabled: bool = True
    seed: int = 0


@dataclass
class FactorizeParams:
    k: int = 2
    n_stages: int = 15
    eta: float = 0.5
    cluster: ClusterParams = field(default_factory=ClusterParams)
    core_min: int = 10
    core_cap: int = 4096
    seed: int = 0

    def to_c(self) -> abi.Params:
        c = self.cluster
        return abi.make_params(
            k=self.k,
            n_stages=self.n_stages,
            eta=self.eta,
            m_target=c.m_target,
            c_min=c.c_min,
            c_max=c.c_max,
            d_max=c.d_max,
            bypass_enabled=c.bypass_enabled,
            core_min=self.core_min,
            core_cap=self.core_cap,
            seed=self.seed,
            cluster_seed=c.seed,
        )


# --------------------------------------------------------------- matrices
class Partition:
    """Ordered clusters of global ids (partition.hpp:19-93)."""

    def __init__(self, clusters: Sequence[Sequence[int]]):
        self.clusters = [np.asarray(c, np.int64) for c in clusters]

    @staticmethod
    def trivial(n: int) -> "Partition":
        return Partition([np.arange(n, dtype=np.int64)])

    @staticmethod
    def single(indices) -> "Partition":
        return Partition([indices])

    def num_clusters(self) -> int:
        return len(self.clusters)

    def size(self) -> int:
        return int(sum(len(c) for c in self.clusters))

    def cluster(self, u: int) -> np.ndarray:
        return self.clusters[u]


class BlockedSparseMatrix:
    """Coordinate data + partition handed to the device as-is.

    ``from_triplets`` keeps the reference semantics (duplicates summed in
    input order, range / finiteness / coverage checks); the checks run on the
    device when ``factorize`` is called.  ``rows/cols/vals`` may be host
    numpy arrays or CUDA torch tensors (device-resident input)."""

    def __init__(self, n: int, rows, cols, vals, partition: Optional[Partition] = None):
        self.n = int(n)
        self.rows, self.cols, self.vals = rows, cols, vals
        self.partition = partition

    @staticmethod
    def from_triplets(n: int, rows, cols, vals, partition: Optional[Partition] = None) -> "BlockedSparseMatrix":
        return BlockedSparseMatrix(n, rows, cols, vals, partition)

    @property
    def on_device(self) -> bool:
        return bool(getattr(self.rows, "is_cuda", False))

    def coo(self, device: int = 0):
        clusters = None
        if self.partition is not None:
            clusters = self.partition.clusters
        return abi.make_coo(self.n, self.rows, self.cols, self.vals, clusters, on_device=self.on_device, device=device)


# ----------------------------------------------------------- factorization
@dataclass
class Rotation:
    indices: np.ndarray
    matrix: np.ndarray
    stage: int


class MmfFactorization(abi.FlatFactorization):
    """``MmfFactorization`` (factorizer.hpp:111-118) in flat arrays, with the
    reference-style accessors on top."""

    def rotations(self, stage: int) -> List[Rotation]:
        st = self.stages[stage]
        return [Rotation(st.rot_indices[t], st.rot_matrices[t], stage + 1) for t in range(len(st.rot_indices))]

    def diagonal_value(self, i: int) -> float:
        pos = np.searchsorted(self.diag_index, i)
        if pos >= len(self.diag_index) or self.diag_index[pos] != i:
            raise IndexError("CoreDiagonal: index not retired")
        return float(self.diag_value[pos])


def _factorize_call(lib, coo, p, h, err, comm: Optional[Communicator]):
    if comm is None:
        return lib.factorize(ctypes.byref(coo), ctypes.byref(p), ctypes.byref(h), err, len(err))
    return lib.lib.pmmf_b200_factorize_sharded(ctypes.byref(coo), ctypes.byref(p), comm.handle, ctypes.byref(h), err,
                                               len(err))


def factorize(matrix: BlockedSparseMatrix, params: FactorizeParams, device: int = 0,
              comm: Optional[Communicator] = None) -> MmfFactorization:
    """pmmf::factorize on the GPU (factorizer.hpp:397-595); with `comm`, the
    clusters of every stage are sharded over its ranks (collective call,
    every rank returns the same factorization)."""
    lib = library()
    coo, keep = matrix.coo(device)
    if matrix.on_device:
        # the library reads the triplets on its own stream: order it after
        # the work that produced them (include/pmmf_b200.h, "Device input")
        import torch

        torch.cuda.current_stream(device).synchronize()
    p = params.to_c()
    h = ctypes.c_void_p()
    err = lib.errbuf()
    abi.raise_for(_factorize_call(lib, coo, p, h, err, comm), err)
    try:
        flat = lib.read_result(h)
    finally:
        lib.result_free(h)
    out = MmfFactorization.__new__(MmfFactorization)
    out.__dict__.update(flat.__dict__)
    out.params = params
    return out


def factorize_handle(matrix: BlockedSparseMatrix, params: FactorizeParams, device: int = 0,
                     comm: Optional[Communicator] = None) -> ctypes.c_void_p:
    """Raw result handle (caller frees with library().result_free)."""
    lib = library()
    coo, keep = matrix.coo(device)
    if matrix.on_device:
        # the library reads the triplets on its own stream: order it after
        # the work that produced them (include/pmmf_b200.h, "Device input")
        import torch

        torch.cuda.current_stream(device).synchronize()
    p = params.to_c()
    h = ctypes.c_void_p()
    err = lib.errbuf()
    abi.raise_for(_factorize_call(lib, coo, p, h, err, comm), err)
    return h


# -------------------------------------------------- factorization container
def save_factorization(handle: ctypes.c_void_p, path: str) -> None:
    """save_factorization (serialize.hpp:167-171): the reference's JSON
    container for a result handle (factorize_handle / load_factorization_handle)."""
    lib = library()
    err = lib.errbuf()
    abi.raise_for(lib.lib.pmmf_b200_result_save(handle, os.fsencode(path), err, len(err)), err)


def load_factorization_handle(path: str) -> ctypes.c_void_p:
    """load_factorization (serialize.hpp:173-183) as a result handle: feeds
    the accessors and MmfOperator (pmmf_b200_operator_create) without
    refactorizing.  The caller frees it with library().result_free."""
    lib = library()
    h = ctypes.c_void_p()
    err = lib.errbuf()
    abi.raise_for(lib.lib.pmmf_b200_result_load(os.fsencode(path), ctypes.byref(h), err, len(err)), err)
    return h


def load_factorization(path: str) -> MmfFactorization:
    lib = library()
    h = load_factorization_handle(path)
    try:
        flat = lib.read_result(h)
        p = abi.Params()
        abi.raise_for(lib.lib.pmmf_b200_result_params(h, ctypes.byref(p)), None)
    finally:
        lib.result_free(h)
    out = MmfFactorization.__new__(MmfFactorization)
    out.__dict__.update(flat.__dict__)
    out.params = FactorizeParams(k=p.k, n_stages=p.n_stages, eta=p.eta, core_min=p.core_min, core_cap=p.core_cap,
                                 seed=p.seed,
                                 cluster=ClusterParams(m_target=p.m_target, c_min=p.c_min, c_max=p.c_max,
                                                       d_max=p.d_max, bypass_enabled=bool(p.bypass_enabled),
                                                       seed=p.cluster_seed))
    return out


def result_handle_from(f: abi.FlatFactorization, params: Optional[FactorizeParams] = None) -> ctypes.c_void_p:
    """A result handle holding an existing factorization (this library's, the
    reference's or a loaded one), for MmfOperator without refactorizing
    (pmmf_b200_result_create / _add_stage / _set_core; PMMF_DATA on
    out-of-range indices).  The caller frees it with library().result_free."""
    lib = library()
    L = lib.lib
    err = lib.errbuf()
    p = params or getattr(f, "params", None) or FactorizeParams(k=int(f.k))
    p = p.to_c() if hasattr(p, "to_c") else p
    p.k = int(f.k)
    h = ctypes.c_void_p()
    abi.raise_for(L.pmmf_b200_result_create(int(f.n), ctypes.byref(p), float(f.residual_sq), ctypes.byref(h), err,
                                            len(err)), err)
    keep = []

    def arr(x, dt):
        a = np.ascontiguousarray(x, dt)
        if a.size == 0:
            a = np.zeros(1, dt)
        keep.append(a)
        return a.ctypes.data

    try:
        for st in f.stages:
            nc = len(st.cluster_offsets) - 1
            abi.raise_for(L.pmmf_b200_result_add_stage(
                h, nc, arr(st.cluster_offsets, np.int64), arr(st.members, np.int64), len(st.rot_indices),
                arr(st.rot_indices, np.int64), arr(st.rot_matrices, np.float64), len(st.elim_index),
                arr(st.elim_index, np.int64), arr(st.elim_diagonal, np.float64), arr(st.elim_off_mass_sq, np.float64),
                len(st.bypassed), arr(st.bypassed, np.int64), err, len(err)), err)
        g = len(f.core_indices)
        abi.raise_for(L.pmmf_b200_result_set_core(
            h, g, arr(f.core_indices, np.int64), arr(f.core, np.float64), len(f.diag_index),
            arr(f.diag_index, np.int64), arr(f.diag_value, np.float64), arr(f.active_history, np.int64),
            len(f.active_history), err, len(err)), err)
    except Exception:
        lib.result_free(h)
        raise
    return h


class MmfOperator:
    """pmmf::MmfOperator (transform_ops.hpp:30-137) on the GPU: wraps a
    factorization (an MmfFactorization / FlatFactorization, or a raw result
    handle) without refactorizing; apply(mode, x) computes Q^T H^(mode) Q x.
    x: one vector (n,) or a batch (b, n), as numpy (host) or a contiguous
    float64 CUDA tensor (device); the result has x's type and shape."""

    class Mode:
        forward, inverse, inv_sqrt = 0, 1, 2

    def __init__(self, f, zero_threshold: float = 1e-12):
        lib = library()
        self._f = f if isinstance(f, abi.FlatFactorization) else None
        own = not isinstance(f, ctypes.c_void_p)
        h = result_handle_from(f) if own else f
        self._op = ctypes.c_void_p()
        err = lib.errbuf()
        try:
            abi.raise_for(lib.operator_create(h, float(zero_threshold), ctypes.byref(self._op), err, len(err)), err)
            s = abi.Summary()
            lib.result_summary(h, ctypes.byref(s))
            self._n = int(s.n)
        finally:
            if own:
                lib.result_free(h)

    def dim(self) -> int:
        return self._n

    def factorization(self):
        if self._f is None:
            raise RuntimeError("MmfOperator was built from a raw handle")
        return self._f

    def inv_sqrt_zeroed_negatives(self) -> int:
        v = ctypes.c_int64()
        library().operator_zeroed_negatives(self._op, ctypes.byref(v))
        return int(v.value)

    def apply_sharded(self, mode: int, x, comm: "Communicator"):
        """apply(mode, x) over the ranks of `comm` (host numpy vectors; every
        rank passes the same x and gets the full result)."""
        lib = library()
        L = lib.lib
        L.pmmf_b200_operator_apply_sharded.restype = ctypes.c_int
        L.pmmf_b200_operator_apply_sharded.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                                       ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                                       ctypes.c_int32, ctypes.c_char_p, ctypes.c_size_t]
        a = np.ascontiguousarray(x, np.float64)
        if a.shape[-1] != self._n or a.ndim > 2:
            raise ValueError("MmfOperator::apply: dimension mismatch")
        out = np.zeros_like(a)
        err = lib.errbuf()
        abi.raise_for(L.pmmf_b200_operator_apply_sharded(self._op, comm.handle, int(mode), 1 if a.ndim == 1 else a.shape[0],
                                                         a.ctypes.data, out.ctypes.data, 0, err, len(err)), err)
        return out

    def apply(self, mode: int, x):
        lib = library()
        err = lib.errbuf()
        if getattr(x, "is_cuda", False):
            import torch

            if x.dtype != torch.float64 or not x.is_contiguous() or x.shape[-1] != self._n:
                raise ValueError("MmfOperator.apply: expected a contiguous float64 (.., n) CUDA tensor")
            out = torch.empty_like(x)
            torch.cuda.current_stream(x.device).synchronize()
            nrhs = 1 if x.dim() == 1 else int(x.shape[0])
            abi.raise_for(lib.operator_apply(self._op, int(mode), nrhs, x.data_ptr(), out.data_ptr(), 1, err,
                                             len(err)), err)
            return out
        a = np.ascontiguousarray(x, np.float64)
        if a.shape[-1] != self._n or a.ndim > 2:
            raise ValueError("MmfOperator::apply: dimension mismatch")
        out = np.zeros_like(a)
        nrhs = 1 if a.ndim == 1 else a.shape[0]
        abi.raise_for(lib.operator_apply(self._op, int(mode), nrhs, a.ctypes.data, out.ctypes.data, 0, err,
                                         len(err)), err)
        return out

    def close(self) -> None:
        if getattr(self, "_op", None):
            library().operator_free(self._op)
            self._op = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def residual_frobenius(handle: ctypes.c_void_p, matrix: "BlockedSparseMatrix", method: str = "dense",
                       cap: int = 4096, device: int = 0) -> float:
    """residual_frobenius (transform_ops.hpp:225-237): "accumulated" =
    sqrt(residual_sq); "dense" = ||A - Q^T H Q||_F reconstructed on the GPU."""
    lib = library()
    coo, keep = matrix.coo(device)
    out = ctypes.c_double()
    err = lib.errbuf()
    st = lib.lib.pmmf_b200_residual_frobenius(handle, ctypes.byref(coo), 0 if method == "accumulated" else 1,
                                              int(cap), ctypes.byref(out), err, len(err))
    abi.raise_for(st, err)
    return out.value


# ------------------------------------------- solver study (solver.hpp)
class PreconditionerKind:
    """PreconditionerKind (solver.hpp:60)."""
    none, jacobi, ssor, ic, pmmf = 0, 1, 2, 3, 4


def preconditioner_name(kind: int) -> str:  # solver.hpp:62-71
    return {0: "none", 1: "jacobi", 2: "ssor", 3: "ic", 4: "pmmf"}.get(int(kind), "?")


class SplitPreconditioner:
    """SplitPreconditioner (solver.hpp:49-52) on the GPU: left(x) = K^-1 x,
    right(x) = K^-T x for one vector (n,) or a batch (b, n) of host vectors."""

    def __init__(self, handle: ctypes.c_void_p, n: int, keep=None):
        self._h = handle
        self._n = int(n)
        self._keep = keep  # e.g. the MmfOperator a pmmf preconditioner wraps

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def _apply(self, side: int, x):
        lib = library()
        a = np.ascontiguousarray(x, np.float64)
        if a.shape[-1] != self._n or a.ndim > 2:
            raise ValueError("SplitPreconditioner: length mismatch")
        out = np.zeros_like(a)
        err = lib.errbuf()
        abi.raise_for(lib.precond_apply(self._h, side, 1 if a.ndim == 1 else a.shape[0], a.ctypes.data,
                                        out.ctypes.data, 0, err, len(err)), err)
        return out

    def left(self, x):
        return self._apply(0, x)

    def right(self, x):
        return self._apply(1, x)

    def info(self):
        k, c, a = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_double()
        library().precond_info(self._h, ctypes.byref(k), ctypes.byref(c), ctypes.byref(a))
        return int(k.value), bool(c.value), float(a.value)

    def close(self) -> None:
        if getattr(self, "_h", None):
            library().precond_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class IncompleteCholesky:
    """IncompleteCholesky (solver.hpp:270-274)."""
    precond: SplitPreconditioner
    compensated: bool = False
    alpha: float = 0.0


def _make_precond(matrix: "BlockedSparseMatrix", kind: int, omega: float, device: int) -> SplitPreconditioner:
    lib = library()
    coo, keep = matrix.coo(device)
    h = ctypes.c_void_p()
    err = lib.errbuf()
    abi.raise_for(lib.precond_create(ctypes.byref(coo), int(kind), float(omega), ctypes.byref(h), err, len(err)), err)
    return SplitPreconditioner(h, matrix.n)


def jacobi_preconditioner(matrix: "BlockedSparseMatrix", device: int = 0) -> SplitPreconditioner:
    """jacobi_preconditioner (solver.hpp:222-233)."""
    return _make_precond(matrix, PreconditionerKind.jacobi, 1.0, device)


def ssor_preconditioner(matrix: "BlockedSparseMatrix", omega: float = 1.0, device: int = 0) -> SplitPreconditioner:
    """ssor_preconditioner (solver.hpp:237-267); omega in (0, 2)."""
    return _make_precond(matrix, PreconditionerKind.ssor, omega, device)


def ic_preconditioner(matrix: "BlockedSparseMatrix", device: int = 0) -> IncompleteCholesky:
    """ic_preconditioner (solver.hpp:278-340): IC(0), one compensated restart."""
    p = _make_precond(matrix, PreconditionerKind.ic, 1.0, device)
    _, comp, alpha = p.info()
    return IncompleteCholesky(p, comp, alpha)


def pmmf_preconditioner(op: "MmfOperator") -> SplitPreconditioner:
    """pmmf_preconditioner (solver.hpp:343-349): K^-1 = K^-T = apply(inv_sqrt)."""
    lib = library()
    h = ctypes.c_void_p()
    err = lib.errbuf()
    abi.raise_for(lib.precond_from_operator(op._op, ctypes.byref(h), err, len(err)), err)
    return SplitPreconditioner(h, op.dim(), keep=op)


@dataclass
class SolveConfig:
    """SolveConfig (solver.hpp:73-86); the preconditioner is passed to
    run_solve_experiment."""
    tol: float = 1e-5
    max_iter: int = 100
    rhs_count: int = 20
    seed: int = 0


@dataclass
class SolveReport:
    """SolveReport (solver.hpp:352-365); runs[r] = (iterations, converged,
    breakdown, residual trace)."""
    method: str
    mean_residual: np.ndarray
    std_residual: np.ndarray
    mean_iterations: float
    max_iterations_used: int
    all_converged: bool
    any_breakdown: bool
    wall_ms_total: float
    per_iteration_ms: float
    iterations: np.ndarray
    converged: np.ndarray
    breakdown: np.ndarray
    residuals: List[np.ndarray]


def run_solve_experiment(matrix: "BlockedSparseMatrix", m: Optional[SplitPreconditioner], cfg: SolveConfig,
                         method_name: str, device: int = 0) -> SolveReport:
    """run_solve_experiment (solver.hpp:368-416): CG / split-preconditioned CG
    on cfg.rhs_count seeded unit-norm right-hand sides, all advanced together
    on the GPU; residual traces aggregated as the reference does."""
    lib = library()
    coo, keep = matrix.coo(device)
    c = abi.SolveConfig(float(cfg.tol), int(cfg.max_iter), int(cfg.rhs_count), int(cfg.seed))
    nr = int(cfg.rhs_count)
    it = np.zeros(nr, np.int32)
    cv = np.zeros(nr, np.int32)
    bk = np.zeros(nr, np.int32)
    tr = np.zeros((nr, int(cfg.max_iter) + 1))
    wall = ctypes.c_double()
    err = lib.errbuf()
    abi.raise_for(lib.solve_precond(ctypes.byref(coo), m.handle if m is not None else None, ctypes.byref(c),
                                    it.ctypes.data_as(abi.c_i32p), cv.ctypes.data_as(abi.c_i32p),
                                    bk.ctypes.data_as(abi.c_i32p), tr.ctypes.data_as(abi.c_f64p), ctypes.byref(wall),
                                    err, len(err)), err)
    runs = [tr[r, : it[r] + 1].copy() for r in range(nr)]
    longest = max(len(x) for x in runs)
    ext = np.array([np.concatenate([x, np.full(longest - len(x), x[-1])]) for x in runs])
    total = int(it.sum())
    return SolveReport(method=method_name, mean_residual=ext.mean(axis=0), std_residual=ext.std(axis=0),
                       mean_iterations=total / nr, max_iterations_used=int(it.max()), all_converged=bool(cv.all()),
                       any_breakdown=bool(bk.any()), wall_ms_total=wall.value,
                       per_iteration_ms=wall.value / total if total else 0.0, iterations=it, converged=cv.astype(bool),
                       breakdown=bk.astype(bool), residuals=runs)


@dataclass
class NystromResult:
    """NystromResult (transform_ops.hpp:252-255)."""
    frobenius_error: float
    columns: np.ndarray


def nystrom_uniform(matrix: "BlockedSparseMatrix", m: int, seed: int, cap: int = 4096,
                    device: int = 0) -> NystromResult:
    """nystrom_uniform (transform_ops.hpp:259-307) evaluated densely on the GPU."""
    lib = library()
    coo, keep = matrix.coo(device)
    fro = ctypes.c_double()
    cols = np.zeros(max(int(m), 1), np.int64)
    err = lib.errbuf()
    abi.raise_for(lib.nystrom_uniform(ctypes.byref(coo), int(m), int(seed), int(cap), ctypes.byref(fro),
                                      cols.ctypes.data_as(abi.c_i64p), err, len(err)), err)
    return NystromResult(fro.value, cols[: int(m)])


# --------------------------------------------------------------- input path
_IO: Optional[abi.IoAbi] = None


def _io() -> abi.IoAbi:
    global _IO
    if _IO is None:
        _IO = abi.IoAbi(library().lib, "pmmf_b200_", device_args=True)
    return _IO


def read_matrix_market(path: str):
    """read_matrix_market (io.hpp:68-129) -> (rows, cols, row, col, val)."""
    rows, cols, r, c, v, _ = _io().read("mm", path)
    return rows, cols, r, c, v


def read_edge_list(path: str):
    """read_edge_list (io.hpp:158-208) -> (n, row, col, val, original_ids)."""
    n, _, r, c, v, ids = _io().read("el", path)
    return n, r, c, v, ids


def write_matrix_market(path: str, rows: int, cols: int, r, c, v) -> None:
    """write_matrix_market (io.hpp:131-147)."""
    _io().write_matrix_market(path, rows, cols, r, c, v)


def laplacian(r, c, v, n: int, shift: float = 0.0, device: int = 0):
    """laplacian (io.hpp:212-228) on the GPU -> (row, col, val), nnz + n entries."""
    return _io().laplacian(r, c, v, n, shift, device)


def symmetrize(r, c, v, device: int = 0):
    """symmetrize (io.hpp:231-250) on the GPU -> (row, col, val)."""
    return _io().symmetrize(r, c, v, device)


# -------------------------------------------------------------- workloads
def _take(w: abi.Workload):
    m = w.nnz
    if m:
        rows = np.ctypeslib.as_array(w.rows, (m,)).copy()
        cols = np.ctypeslib.as_array(w.cols, (m,)).copy()
        vals = np.ctypeslib.as_array(w.vals, (m,)).copy()
    else:
        rows = np.zeros(0, np.int64)
        cols = np.zeros(0, np.int64)
        vals = np.zeros(0, np.float64)
    n = w.n
    library().lib.pmmf_b200_workload_free(ctypes.byref(w))
    return n, rows, cols, vals


def workload_rmat(scale: int, edges_per_vertex: int, seed: int = 42, shift: float = 1e-2):
    w = abi.Workload()
    rc = library().lib.pmmf_b200_workload_rmat(
        ctypes.c_int32(scale), ctypes.c_int32(edges_per_vertex), ctypes.c_uint64(seed), ctypes.c_double(shift), ctypes.byref(w)
    )
    if rc:
        raise ValueError("workload_rmat: bad arguments")
    return _take(w)


def workload_dense_spd(n: int, d: int, seed: int = 42, shift: float = 1e-3):
    w = abi.Workload()
    rc = library().lib.pmmf_b200_workload_dense_spd(ctypes.c_int64(n), ctypes.c_int64(d), ctypes.c_uint64(seed), ctypes.c_double(shift), ctypes.byref(w))
    if rc:
        raise ValueError("workload_dense_spd: bad arguments")
    return _take(w)


def workload_rbf(n: int, dim: int = 10, bandwidth: float = 0.5, seed: int = 42, shift: float = 1e-4):
    w = abi.Workload()
    rc = library().lib.pmmf_b200_workload_rbf(
        ctypes.c_int64(n), ctypes.c_int32(dim), ctypes.c_double(bandwidth), ctypes.c_uint64(seed), ctypes.c_double(shift), ctypes.byref(w)
    )
    if rc:
        raise ValueError("workload_rbf: bad arguments")
    return _take(w)


def workload_aniso_grid(side: int, ax: float = 100.0, ay: float = 1.0):
    w = abi.Workload()
    rc = library().lib.pmmf_b200_workload_aniso_grid(ctypes.c_int64(side), ctypes.c_double(ax), ctypes.c_double(ay), ctypes.byref(w))
    if rc:
        raise ValueError("workload_aniso_grid: bad arguments")
    return _take(w)
