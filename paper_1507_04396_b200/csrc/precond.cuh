// precond.cuh — split preconditioners M = K K^T (solver.hpp:46-56) as the
// CG harness and the C-ABI see them.
#pragma once

#include <memory>

#include "common.cuh"

namespace pmmf_b200 {

// The pair (K^-1, K^-T) of SplitPreconditioner (solver.hpp:49-52) on the
// device: vectors are index-major n x nr (v[i * nr + r], i a global id).
// The handle owns a stream: its long-lived buffers are allocated and
// released on it (it is destroyed last, after the derived members).
struct SplitPrecond {
  cudaStream_t own = nullptr;
  int kind = PMMF_PRECOND_NONE;
  i64 n = 0;
  int device = 0;
  int compensated = 0;  // IncompleteCholesky (solver.hpp:270-274)
  double alpha = 0.0;
  SplitPrecond() { PMMF_CUDA(cudaStreamCreateWithFlags(&own, cudaStreamNonBlocking)); }
  SplitPrecond(const SplitPrecond&) = delete;
  SplitPrecond& operator=(const SplitPrecond&) = delete;
  virtual ~SplitPrecond() {
    if (own) {
      cudaStreamSynchronize(own);
      cudaStreamDestroy(own);
    }
  }
  // out = K^-1 in (side 0) or K^-T in (side 1); in and out are distinct.
  virtual void apply(int side, int nr, const double* in, double* out, cudaStream_t s) = 0;
};

// jacobi / ssor / ic (precond.cu).
std::unique_ptr<SplitPrecond> make_precond(const pmmf_b200_coo* a, int kind, double omega);
// pmmf_preconditioner (operator.cu): wraps an Operator handle.
std::unique_ptr<SplitPrecond> precond_from_operator(void* op);
// jacobi_eigensystem (dense.hpp:191-199) of a row-major g x g device
// matrix; vectors(i, e) row-major (operator.cu).
void eigensystem_dev(int g, const double* a, double* values, double* vectors, cudaStream_t s);
// run_solve_experiment over pcg_symmetric with pc (nullptr = plain CG).
void run_cg(const pmmf_b200_coo* a, SplitPrecond* pc, const pmmf_b200_solve_config* cfg, int32_t* iterations,
            int32_t* converged, int32_t* breakdown, double* residuals, double* wall_ms);

}  // namespace pmmf_b200
