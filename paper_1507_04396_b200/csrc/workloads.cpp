// workloads.cpp — seeded synthetic inputs for the BASELINE.json configs.
//
// The reference ships no R-MAT / RBF / anisotropic generators (SURVEY.md
// Appendix B, graphs.hpp); these follow the exact recipes of SURVEY.md §8(d)
// with the reference's Rng stream (rng.hpp), so the GPU path and the CPU
// oracles consume identical triplets.  Output is COO in emission order.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <utility>
#include <vector>

#include "../../include/pmmf_b200_workloads.h"
#include "recipes.hpp"
#include "rng.cuh"

using pmmf_b200::Xoshiro;

namespace {

// The recipes consume draws through the reference's interface (rng.hpp:53-71).
struct Source {
  Xoshiro r;
  explicit Source(uint64_t seed) : r(seed) {}
  double uniform01() { return r.uniform01(); }
  double normal() { return pmmf_b200::normal_draw(r); }
};

int emit(const pmmf_recipes::Coo& coo, pmmf_b200_workload* out) {
  out->n = coo.n;
  out->nnz = static_cast<int64_t>(coo.v.size());
  const std::size_t m = coo.v.size();
  out->rows = static_cast<int64_t*>(std::malloc(std::max<std::size_t>(1, m) * sizeof(int64_t)));
  out->cols = static_cast<int64_t*>(std::malloc(std::max<std::size_t>(1, m) * sizeof(int64_t)));
  out->vals = static_cast<double*>(std::malloc(std::max<std::size_t>(1, m) * sizeof(double)));
  if (!out->rows || !out->cols || !out->vals) return 1;
  if (m) {
    std::memcpy(out->rows, coo.r.data(), m * sizeof(int64_t));
    std::memcpy(out->cols, coo.c.data(), m * sizeof(int64_t));
    std::memcpy(out->vals, coo.v.data(), m * sizeof(double));
  }
  return 0;
}

}  // namespace

extern "C" {

// R-MAT graph, normalized Laplacian + shift·I (SURVEY.md §8(d) "R-MAT").
int pmmf_b200_workload_rmat(int32_t scale, int32_t edges_per_vertex, uint64_t seed, double shift,
                            pmmf_b200_workload* out) {
  Source rng(seed);
  pmmf_recipes::Coo coo;
  if (!pmmf_recipes::rmat(scale, edges_per_vertex, rng, shift, coo)) return 1;
  return emit(coo, out);
}

// Dense SPD A = X X^T / d + shift·I, X n x d ~ N(0,1) row-major (config 1).
int pmmf_b200_workload_dense_spd(int64_t n, int64_t d, uint64_t seed, double shift,
                                 pmmf_b200_workload* out) {
  Source rng(seed);
  pmmf_recipes::Coo coo;
  if (!pmmf_recipes::dense_spd(n, d, rng, shift, coo)) return 1;
  return emit(coo, out);
}

// Gaussian RBF kernel on n uniform points in [0,1]^dim (config 3).
int pmmf_b200_workload_rbf(int64_t n, int32_t dim, double bandwidth, uint64_t seed, double shift,
                           pmmf_b200_workload* out) {
  Source rng(seed);
  pmmf_recipes::Coo coo;
  if (!pmmf_recipes::rbf(n, dim, bandwidth, rng, shift, coo)) return 1;
  return emit(coo, out);
}

// 5-point anisotropic Poisson on a side x side grid (config 5).
int pmmf_b200_workload_aniso_grid(int64_t side, double ax, double ay, pmmf_b200_workload* out) {
  pmmf_recipes::Coo coo;
  if (!pmmf_recipes::aniso_grid(side, ax, ay, coo)) return 1;
  return emit(coo, out);
}

// Unit-norm Gaussian right-hand sides of run_solve_experiment
// (solver.hpp:375-381): rhs r from Rng(derive(seed, {0xB0, r})).normal().
int pmmf_b200_workload_rhs(int64_t n, int32_t count, uint64_t seed, double* out) {
  for (int32_t r = 0; r < count; ++r) {
    const uint64_t path[2] = {0xB0u, static_cast<uint64_t>(r)};
    Xoshiro rng(pmmf_b200::derive(seed, path));
    double* b = out + static_cast<int64_t>(r) * n;
    for (int64_t i = 0; i < n; ++i) b[i] = pmmf_b200::normal_draw(rng);
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += b[i] * b[i];
    const double norm = std::sqrt(s);
    if (norm > 0.0)
      for (int64_t i = 0; i < n; ++i) b[i] /= norm;
  }
  return 0;
}

void pmmf_b200_workload_free(pmmf_b200_workload* w) {
  if (!w) return;
  std::free(w->rows);
  std::free(w->cols);
  std::free(w->vals);
  w->rows = w->cols = nullptr;
  w->vals = nullptr;
}

}  // extern "C"
