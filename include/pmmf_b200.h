/*
 * pmmf_b200.h — C-ABI of the B200-native pMMF stage loop.
 *
 * This is the drop-in boundary: plain pointers and sizes, no torch or C++
 * types.  Each entry point replaces one reference interface of
 * /root/reference/proj/include/pmmf (cited per function).  The C++ shim in
 * include/pmmf_b200/dropin.hpp and the Python mirror in
 * paper_1507_04396_b200/api.py are thin layers over these calls.
 *
 * Conventions
 *   - every call returns a pmmf_b200_status; on failure a NUL-terminated
 *     message is written to err[0..errlen) when err != NULL.  The status
 *     maps 1:1 onto the reference's exception types (types.hpp:24-32,
 *     factorizer.hpp:44-50, :404-408, :573-576, blocked_matrix.hpp:143-149).
 *   - indices are int64 global ids (types.hpp:11 `index_t`), values fp64.
 *   - dense k x k rotation blocks and the g x g core are row-major, like
 *     pmmf::DenseMatrix (dense.hpp:36).
 *   - multi right-hand-side vectors are stored rhs-major: rhs r occupies
 *     [r*n, (r+1)*n).
 */
#ifndef PMMF_B200_H
#define PMMF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum pmmf_b200_status {
  PMMF_OK = 0,
  PMMF_INVALID_ARGUMENT = 1, /* std::invalid_argument               */
  PMMF_OUT_OF_RANGE = 2,     /* std::out_of_range                   */
  PMMF_NUMERIC = 3,          /* pmmf::NumericError                  */
  PMMF_DATA = 4,             /* pmmf::DataError                     */
  PMMF_CUDA = 5,             /* device / driver failure             */
  PMMF_INTERNAL = 6          /* anything else (bug)                 */
} pmmf_b200_status;

/* FactorizeParams (factorizer.hpp:35-51) with its nested ClusterParams
 * (clustering.hpp:28-41).  cluster.seed is accepted but, as in the
 * reference (factorizer.hpp:435-436), re-derived per stage. */
typedef struct pmmf_b200_params {
  int32_t k;              /* rotation order, 2 = Givens                 */
  int32_t n_stages;       /* P                                          */
  double eta;             /* rotations per cluster: floor(eta * c)      */
  int64_t m_target;       /* m                                          */
  int64_t c_min;
  int64_t c_max;
  int32_t d_max;          /* D_max                                      */
  int32_t bypass_enabled;
  uint64_t cluster_seed;  /* ignored (re-derived per stage)             */
  int64_t core_min;
  int64_t core_cap;
  uint64_t seed;
} pmmf_b200_params;

/* Input matrix in coordinate form plus its block partition: the data of
 * BlockedSparseMatrix::from_triplets(n, entries, partition)
 * (blocked_matrix.hpp:133-156).  n_clusters == 0 means Partition::trivial(n)
 * (partition.hpp:57-61).  Duplicates are summed in input order.
 *
 * Device input (on_device != 0): rows/cols/vals must be CUDA pointers on
 * `device`.  The library reads them on its own non-blocking stream, so the
 * caller must have COMPLETED the work that produced them before the call
 * (e.g. cudaStreamSynchronize on the producing stream); the Python layer
 * does this for torch tensors.  Every entry point that takes device
 * buffers returns only after its device outputs are complete. */
typedef struct pmmf_b200_coo {
  int64_t n;
  int64_t nnz;
  const int64_t* rows;
  const int64_t* cols;
  const double* vals;
  int64_t n_clusters;
  const int64_t* cluster_offsets; /* n_clusters + 1 entries           */
  const int64_t* cluster_members; /* cluster_offsets[n_clusters] ids  */
  int32_t on_device;              /* rows/cols/vals are CUDA pointers */
  int32_t device;                 /* CUDA ordinal for the computation */
} pmmf_b200_coo;

/* Scalar view of MmfFactorization (factorizer.hpp:111-118) and
 * FactorizeStats::trivial (:105-109). */
typedef struct pmmf_b200_summary {
  int64_t n;
  int64_t n_stages;
  int64_t k;
  int64_t core_size;      /* |h.core_indices|                            */
  int64_t n_diagonal;     /* |h.diagonal|                                */
  int64_t trivial;
  double residual_sq;
} pmmf_b200_summary;

/* Sizes of one Stage (factorizer.hpp:65-70). */
typedef struct pmmf_b200_stage_sizes {
  int64_t n_clusters;     /* stage partition, bypass cluster included */
  int64_t partition_size;
  int64_t n_rotations;
  int64_t n_eliminated;
  int64_t n_bypassed;
} pmmf_b200_stage_sizes;

/* SolveConfig (solver.hpp:73-86); the preconditioner is chosen by passing
 * an operator (pmmf) or NULL (none) to pmmf_b200_solve. */
typedef struct pmmf_b200_solve_config {
  double tol;
  int32_t max_iter;
  int32_t rhs_count;
  uint64_t seed;
} pmmf_b200_solve_config;

/* ---- factorization: pmmf::factorize (factorizer.hpp:397-595) -------- */

/* Runs the stage loop on the GPU given by a->device.  *out receives an
 * opaque result handle (free with pmmf_b200_result_free). */
int pmmf_b200_factorize(const pmmf_b200_coo* a, const pmmf_b200_params* p, void** out,
                        char* err, size_t errlen);

/* MmfFactorization scalars. */
int pmmf_b200_result_summary(void* h, pmmf_b200_summary* out);
/* f.active_history (factorizer.hpp:116): n_stages + 1 entries. */
int pmmf_b200_result_active_history(void* h, int64_t* out);
/* f.stages[s] sizes and contents.  Rotations are cluster-major
 * (factorizer.hpp:67): rot_indices is n_rotations x k, rot_matrices is
 * n_rotations x k x k row-major.  Eliminations in stage order (:68). */
int pmmf_b200_result_stage_sizes(void* h, int64_t s, pmmf_b200_stage_sizes* out);
int pmmf_b200_result_stage(void* h, int64_t s, int64_t* cluster_offsets, int64_t* members,
                           int64_t* rot_indices, double* rot_matrices, int64_t* elim_index,
                           double* elim_diagonal, double* elim_off_mass_sq, int64_t* bypassed);
/* f.h (CoreDiagonal, factorizer.hpp:72-84): core_indices ascending,
 * core g x g row-major, retired diagonal ascending by index. */
int pmmf_b200_result_core(void* h, int64_t* core_indices, double* core, int64_t* diag_index,
                          double* diag_value);
/* FactorizeStats (factorizer.hpp:86-109): phases = {clustering, gram,
 * rotations, apply, reblocking, total} in ms; stage_info is n_stages x 7
 * {stage, clusters, bypassed, rotations, eliminated, active_after, depth}. */
int pmmf_b200_result_stats(void* h, double* phases, int64_t* stage_info);
void pmmf_b200_result_free(void* h);

/* ---- factorization container: save_factorization / load_factorization
 * (serialize.hpp:167-183), the reference's versioned JSON schema
 * ("pmmf-factorization", version 1, serialize.hpp:61-165) written and read
 * without a JSON library.  Doubles round-trip exactly.  A loaded handle
 * serves every pmmf_b200_result_* accessor and pmmf_b200_operator_create
 * (MmfOperator without refactorizing); its stats are empty.  Errors:
 * PMMF_DATA (DataError: unreadable file, unknown format or version, size
 * mismatches). */
int pmmf_b200_result_save(void* h, const char* path, char* err, size_t errlen);
int pmmf_b200_result_load(const char* path, void** out, char* err, size_t errlen);
/* MmfFactorization::params (factorizer.hpp:117). */
int pmmf_b200_result_params(void* h, pmmf_b200_params* out);

/* ---- building a result handle from an existing MmfFactorization ------
 * (the data of factorizer.hpp:56-118 in the accessors' flat layout), so
 * that a factorization made elsewhere (the reference's pmmf::factorize, a
 * file) can drive pmmf_b200_operator_create: the counterpart of
 * MmfOperator(shared_ptr<const MmfFactorization>, zero_threshold)
 * (transform_ops.hpp:32-41).  Create, add every stage in order, set the
 * core; the handle is validated (PMMF_DATA on an index outside [0, n), a
 * rotation order other than params->k, k outside [2, 8], inconsistent
 * offsets) when the core is set.  Free with pmmf_b200_result_free. */
int pmmf_b200_result_create(int64_t n, const pmmf_b200_params* params, double residual_sq, void** out, char* err,
                            size_t errlen);
int pmmf_b200_result_add_stage(void* h, int64_t n_clusters, const int64_t* cluster_offsets, const int64_t* members,
                               int64_t n_rotations, const int64_t* rot_indices, const double* rot_matrices,
                               int64_t n_eliminated, const int64_t* elim_index, const double* elim_diagonal,
                               const double* elim_off_mass_sq, int64_t n_bypassed, const int64_t* bypassed,
                               char* err, size_t errlen);
int pmmf_b200_result_set_core(void* h, int64_t g, const int64_t* core_indices, const double* core,
                              int64_t n_diagonal, const int64_t* diag_index, const double* diag_value,
                              const int64_t* active_history, int64_t n_history, char* err, size_t errlen);

/* ---- multi-GPU: the clusters of every stage sharded over ranks -------
 * (replaces the reference's fork-join thread pool over
 * the clusters of a stage, parallel.hpp:25-71 as used at
 * factorizer.hpp:494-504 and :513).  One process per GPU: rank 0 makes a
 * unique id, the launcher shares it (e.g. torch.distributed), every rank
 * creates its communicator and calls pmmf_b200_factorize_sharded
 * collectively.  Every rank returns the same, complete factorization,
 * bit-identical to pmmf_b200_factorize for any number of ranks. */
#define PMMF_B200_COMM_ID_BYTES 128
int pmmf_b200_comm_unique_id(uint8_t* id, char* err, size_t errlen);
/* NCCL communicator over nranks processes (nranks == 1 may pass id = NULL;
 * its exchanges then run as self-broadcasts). */
int pmmf_b200_comm_create(int32_t nranks, int32_t rank, const uint8_t* id, int32_t device, void** comm,
                          char* err, size_t errlen);
/* nranks virtual ranks run one after another in this process on one GPU
 * (test hook: proves the decomposition bit-exact on a single device). */
int pmmf_b200_comm_create_virtual(int32_t nranks, int32_t device, void** comm, char* err, size_t errlen);
void pmmf_b200_comm_free(void* comm);
/* pmmf::factorize with the stage's clusters split over the communicator's
 * ranks (a->device must be the communicator's device). */
int pmmf_b200_factorize_sharded(const pmmf_b200_coo* a, const pmmf_b200_params* p, void* comm, void** out,
                                char* err, size_t errlen);
/* The cluster split (host only): contiguous ranges lo[0..nranks] of about
 * equal cost c_u^2 + 64 nnz_u (nnz may be NULL). */
int pmmf_b200_shard_ranges(int64_t nclusters, const int64_t* sizes, const int64_t* nnz, int32_t nranks,
                           int64_t* lo);

/* ---- MmfOperator (transform_ops.hpp:30-137) ------------------------- */

enum { PMMF_APPLY_FORWARD = 0, PMMF_APPLY_INVERSE = 1, PMMF_APPLY_INV_SQRT = 2 };

/* Builds the operator for a factorization (core eigensystem,
 * transform_ops.hpp:34-41).  The result handle may be freed afterwards. */
int pmmf_b200_operator_create(void* result, double zero_threshold, void** op, char* err,
                              size_t errlen);
/* out = Q^T H^(mode) Q in for nrhs vectors (transform_ops.hpp:51-67).
 * in/out are host pointers unless on_device != 0. */
int pmmf_b200_operator_apply(void* op, int32_t mode, int64_t nrhs, const double* in,
                             double* out, int32_t on_device, char* err, size_t errlen);
/* The same apply over the ranks of a communicator (pmmf_b200_comm_*,
 * SURVEY.md §8(e) "MMF apply: shard by cluster per stage"): called
 * collectively, every rank passes the same input vectors and receives the
 * full result.  Per stage each rank applies the rotations of its range of
 * apply groups; the updated rows are exchanged before the next stage.
 * Bit-identical to pmmf_b200_operator_apply for any rank count. */
int pmmf_b200_operator_apply_sharded(void* op, void* comm, int32_t mode, int64_t nrhs, const double* in,
                                     double* out, int32_t on_device, char* err, size_t errlen);
/* residual_frobenius (transform_ops.hpp:225-237): method 0 = accumulated
 * (sqrt(residual_sq)), 1 = dense ||A - Q^T H Q||_F with the reconstruction
 * on the GPU (reconstruct_dense, :175-213; PMMF_NUMERIC when n > cap, as
 * the reference).  The dense value equals the reference's up to rounding
 * (it reconstructs by the apply's level order). */
int pmmf_b200_residual_frobenius(void* result, const pmmf_b200_coo* a, int32_t method, int64_t cap, double* out,
                                 char* err, size_t errlen);
/* inv_sqrt_zeroed_negatives() (transform_ops.hpp:47-49). */
int pmmf_b200_operator_zeroed_negatives(void* op, int64_t* out);
void pmmf_b200_operator_free(void* op);

/* ---- solver: run_solve_experiment (solver.hpp:368-416) -------------- */

/* Split-preconditioned CG (pcg_symmetric, solver.hpp:112-167) with
 * K^-1 = K^-T = op->apply(inv_sqrt) (pmmf_preconditioner, :343-349), or
 * plain CG when op == NULL (solver.hpp:170-).  All rhs_count right-hand
 * sides are solved together.  Outputs: iterations/converged/breakdown per
 * rhs; residuals is rhs_count x (max_iter + 1), residuals[r][it] =
 * ||b - A x_it|| (NaN past the end of run r); wall_ms = total. */
int pmmf_b200_solve(const pmmf_b200_coo* a, void* op, const pmmf_b200_solve_config* cfg,
                    int32_t* iterations, int32_t* converged, int32_t* breakdown, double* residuals,
                    double* wall_ms, char* err, size_t errlen);

/* ---- dense Gram mode (gram_of_cluster_sparse, blocked_matrix.hpp:238-254) */

/* Process-wide choice of the dense-cluster Gram kernel.  0 (default): the
 * bitwise SIMT SYRK, every G[a][b] summed over the rows in the reference's
 * order with separately rounded products.  1: FP64 tensor cores (DMMA
 * mma.sync m8n8k4, operands staged by TMA): G agrees to ~1e-15 relative,
 * not bitwise, so a pivot whose score margin is within that distance can
 * differ from the reference (the near-tie clause of the parity contract).
 * Also PMMF_B200_GRAM_DMMA=1 at load time.  Returns PMMF_INVALID_ARGUMENT
 * for another mode. */
int pmmf_b200_set_dense_gram(int32_t mode);
int32_t pmmf_b200_get_dense_gram(void);

/* ---- comparison preconditioners (solver.hpp:46-56, :224-349) -------- */

/* PreconditionerKind (solver.hpp:60).  A preconditioner handle is a split
 * pair M = K K^T given by the actions of K^-1 (side 0, "left") and K^-T
 * (side 1, "right"), built on the GPU of a->device from the same triplets
 * (and input partition) a factorization takes:
 *   JACOBI  jacobi_preconditioner (solver.hpp:222-233): 1/sqrt(a_ii), 0 for
 *           a_ii <= 0;
 *   SSOR    ssor_preconditioner (:237-267), omega in (0, 2), else
 *           PMMF_INVALID_ARGUMENT; a zero diagonal entry is PMMF_NUMERIC;
 *   IC      ic_preconditioner (:278-340): IC(0) on the pattern of the lower
 *           triangle (stored zeros included), restarted once on
 *           A + alpha diag(A) after a breakdown; PMMF_NUMERIC when that is
 *           impossible or breaks down again.
 * The triangular solves and the IC(0) factorization are bit-identical to
 * the reference's sequential loops (same operation order per entry). */
enum { PMMF_PRECOND_NONE = 0, PMMF_PRECOND_JACOBI = 1, PMMF_PRECOND_SSOR = 2, PMMF_PRECOND_IC = 3,
       PMMF_PRECOND_PMMF = 4 };
int pmmf_b200_precond_create(const pmmf_b200_coo* a, int32_t kind, double omega, void** out, char* err,
                             size_t errlen);
/* pmmf_preconditioner (solver.hpp:343-349): K^-1 = K^-T = op->apply(inv_sqrt).
 * The operator handle must outlive the preconditioner. */
int pmmf_b200_precond_from_operator(void* op, void** out, char* err, size_t errlen);
/* out = K^-1 in (side 0) or K^-T in (side 1) for nrhs rhs-major vectors;
 * host pointers unless on_device != 0 (then device pointers on the
 * preconditioner's GPU, ordered after the caller's prior work by a device
 * synchronisation). */
int pmmf_b200_precond_apply(void* pc, int32_t side, int64_t nrhs, const double* in, double* out,
                            int32_t on_device, char* err, size_t errlen);
/* IncompleteCholesky::{compensated, alpha} (solver.hpp:270-274); 0 / 0.0
 * for the other kinds. */
int pmmf_b200_precond_info(void* pc, int32_t* kind, int32_t* compensated, double* alpha);
void pmmf_b200_precond_free(void* pc);
/* run_solve_experiment with any split preconditioner (pc == NULL: plain CG,
 * solver.hpp:170-172); outputs as pmmf_b200_solve. */
int pmmf_b200_solve_precond(const pmmf_b200_coo* a, void* pc, const pmmf_b200_solve_config* cfg,
                            int32_t* iterations, int32_t* converged, int32_t* breakdown, double* residuals,
                            double* wall_ms, char* err, size_t errlen);

/* ---- Nystrom sketch: nystrom_uniform (transform_ops.hpp:252-307) ----- */

/* m distinct columns drawn uniformly by Rng(seed) (partial Fisher-Yates),
 * A ~= C W^+ C^T with W^+ from the Jacobi eigensystem of W (eigenvalues
 * |l| <= 1e-10 max|l| dropped), evaluated densely on the GPU.  Writes
 * ||A - C W^+ C^T||_F and the m sampled columns (ascending).  m outside
 * [1, n] is PMMF_INVALID_ARGUMENT, n > cap PMMF_NUMERIC (as the reference).
 * Every entry and the final sum follow the reference's operation order. */
int pmmf_b200_nystrom_uniform(const pmmf_b200_coo* a, int64_t m, uint64_t seed, int64_t cap,
                              double* frobenius_error, int64_t* columns, char* err, size_t errlen);

/* ---- input path (io.hpp:27-250) -------------------------------------- */

/* TripletMatrix (io.hpp:27-33) / EdgeList (io.hpp:150-154), owned by the
 * library (free with pmmf_b200_triplets_free).  For an edge list rows =
 * cols = the compacted node count and original_ids[new] = id in the file;
 * for Matrix Market original_ids is NULL. */
typedef struct pmmf_b200_triplets {
  int64_t rows;
  int64_t cols;
  int64_t nnz;
  int64_t* row;
  int64_t* col;
  double* val;
  int64_t n_ids;
  int64_t* original_ids;
} pmmf_b200_triplets;
/* read_matrix_market (io.hpp:68-129): coordinate real/integer/pattern,
 * general/symmetric; symmetric files mirror off-diagonal entries, pattern
 * entries get 1, indices become 0-based.  PMMF_DATA on malformed input. */
int pmmf_b200_read_matrix_market(const char* path, pmmf_b200_triplets** out, char* err, size_t errlen);
/* read_edge_list (io.hpp:158-208): "u v [w]" lines, '#' comments, weight 1
 * when absent, self-loops kept once, ids compacted in ascending order. */
int pmmf_b200_read_edge_list(const char* path, pmmf_b200_triplets** out, char* err, size_t errlen);
void pmmf_b200_triplets_free(pmmf_b200_triplets* t);
/* write_matrix_market (io.hpp:131-147): general real, %.17g values. */
int pmmf_b200_write_matrix_market(const char* path, int64_t rows, int64_t cols, int64_t nnz, const int64_t* r,
                                  const int64_t* c, const double* v, char* err, size_t errlen);
/* laplacian (io.hpp:212-228) on the GPU: out = the adjacency negated in
 * input order, then (i, i, degree_i + shift) for i < n; out arrays hold
 * nnz + n entries.  Degrees are the reference's sequential sums (input
 * order), bit for bit.  Pointers are device pointers when on_device. */
int pmmf_b200_laplacian(int64_t n, int64_t nnz, const int64_t* r, const int64_t* c, const double* v, double shift,
                        int32_t on_device, int32_t device, int64_t* out_r, int64_t* out_c, double* out_v, char* err,
                        size_t errlen);
/* symmetrize (io.hpp:231-250) on the GPU: A + A^T, each unordered pair
 * summed once in input order, emitted in (min, max) order as (i,j),(j,i),
 * diagonal doubled.  Out arrays need room for 2 nnz entries; *out_nnz
 * receives the count. */
int pmmf_b200_symmetrize(int64_t nnz, const int64_t* r, const int64_t* c, const double* v, int32_t on_device,
                         int32_t device, int64_t* out_nnz, int64_t* out_r, int64_t* out_c, double* out_v, char* err,
                         size_t errlen);

/* ---- misc ----------------------------------------------------------- */

/* rotation_from_gram (factorizer.hpp:150-171) on one k x k row-major
 * block; host-side helper used for the known-answer tests. */
int pmmf_b200_rotation_from_gram(int32_t k, const double* g, double* q, char* err, size_t errlen);

/* Number of CUDA kernels this library launched since load (evidence for
 * bench.py's gpu_launches).  Counts every launch site in csrc/. */
int64_t pmmf_b200_kernel_launches(void);

/* Live kernel accounting for benchmarks: when enabled, instrumented launch
 * sites ("rotate_write", "rotate_count", ...) bracket their kernels with CUDA
 * events on the launching stream and accumulate device time and algorithmic
 * bytes.  Enabling resets the counters. */
void pmmf_b200_profile_enable(int32_t on);
int pmmf_b200_profile_read(const char* name, int64_t* launches, double* ms, double* bytes);

/* Device memory kept between calls: the library allocates from its own
 * stream-ordered memory pool per device (never the device's default pool,
 * whose attributes stay the caller's), keeps freed pool memory mapped, and
 * caches whole large blocks (>= 32 MB) for reuse by later factorizations
 * (mapping fresh memory costs ~80 ms per GB).  Returns the cached bytes on `device`; with release != 0
 * the cache is returned to the device pool and the pool trimmed first
 * (returns 0 then).  Blocks in use are never affected. */
int64_t pmmf_b200_cached_bytes(int32_t device, int32_t release);

/* Library version string. */
const char* pmmf_b200_version(void);

#ifdef __cplusplus
}
#endif

#endif /* PMMF_B200_H */
