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
#include "rng.cuh"

using pmmf_b200::Xoshiro;

namespace {

struct Coo {
  std::vector<int64_t> r, c;
  std::vector<double> v;
  void push(int64_t i, int64_t j, double x) {
    r.push_back(i);
    c.push_back(j);
    v.push_back(x);
  }
};

int emit(Coo& coo, int64_t n, pmmf_b200_workload* out) {
  out->n = n;
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
  if (scale < 1 || scale > 30 || edges_per_vertex < 1) return 1;
  const int64_t n = int64_t{1} << scale;
  Xoshiro rng(seed);
  const int64_t samples = (static_cast<int64_t>(edges_per_vertex) * n) / 2;
  const double a = 0.57, b = 0.19, c = 0.19;
  const double ab = a + b, abc = a + b + c;
  std::vector<uint64_t> edges;
  edges.reserve(static_cast<std::size_t>(samples));
  for (int64_t e = 0; e < samples; ++e) {
    int64_t i = 0, j = 0;
    for (int l = 0; l < scale; ++l) {
      const double r = rng.uniform01();
      const int q = r < a ? 0 : (r < ab ? 1 : (r < abc ? 2 : 3));
      i = 2 * i + (q >> 1);
      j = 2 * j + (q & 1);
    }
    if (i == j) continue;
    const int64_t lo = std::min(i, j), hi = std::max(i, j);
    edges.push_back((static_cast<uint64_t>(lo) << 32) | static_cast<uint64_t>(hi));
  }
  std::sort(edges.begin(), edges.end());
  edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
  std::vector<int64_t> deg(static_cast<std::size_t>(n), 0);
  for (uint64_t e : edges) {
    ++deg[e >> 32];
    ++deg[e & 0xffffffffull];
  }
  Coo coo;
  coo.r.reserve(2 * edges.size() + n);
  coo.c.reserve(2 * edges.size() + n);
  coo.v.reserve(2 * edges.size() + n);
  for (uint64_t e : edges) {
    const int64_t i = static_cast<int64_t>(e >> 32), j = static_cast<int64_t>(e & 0xffffffffull);
    const double w = -1.0 / std::sqrt(static_cast<double>(deg[i]) * static_cast<double>(deg[j]));
    coo.push(i, j, w);
    coo.push(j, i, w);
  }
  for (int64_t i = 0; i < n; ++i) coo.push(i, i, (deg[i] > 0 ? 1.0 : 0.0) + shift);
  return emit(coo, n, out);
}

// Dense SPD A = X X^T / d + shift·I, X n x d ~ N(0,1) row-major (config 1).
int pmmf_b200_workload_dense_spd(int64_t n, int64_t d, uint64_t seed, double shift,
                                 pmmf_b200_workload* out) {
  if (n < 1 || d < 1) return 1;
  Xoshiro rng(seed);
  std::vector<double> x(static_cast<std::size_t>(n * d));
  for (auto& v : x) v = pmmf_b200::normal_draw(rng);
  Coo coo;
  coo.r.reserve(n * n);
  coo.c.reserve(n * n);
  coo.v.reserve(n * n);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double s = 0.0;
      for (int64_t t = 0; t < d; ++t) s += x[i * d + t] * x[j * d + t];
      s /= static_cast<double>(d);
      if (i == j) s += shift;
      coo.push(i, j, s);
    }
  return emit(coo, n, out);
}

// Gaussian RBF kernel on n uniform points in [0,1]^dim (config 3):
// K_ij = exp(-|x_i - x_j|^2 / (2 bw^2)) + shift·delta_ij.
int pmmf_b200_workload_rbf(int64_t n, int32_t dim, double bandwidth, uint64_t seed, double shift,
                           pmmf_b200_workload* out) {
  if (n < 1 || dim < 1) return 1;
  Xoshiro rng(seed);
  std::vector<double> x(static_cast<std::size_t>(n * dim));
  for (auto& v : x) v = rng.uniform01();
  const double denom = 2.0 * bandwidth * bandwidth;
  Coo coo;
  coo.r.reserve(n * n);
  coo.c.reserve(n * n);
  coo.v.reserve(n * n);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double d2 = 0.0;
      for (int t = 0; t < dim; ++t) {
        const double df = x[i * dim + t] - x[j * dim + t];
        d2 += df * df;
      }
      double k = std::exp(-d2 / denom);
      if (i == j) k += shift;
      coo.push(i, j, k);
    }
  return emit(coo, n, out);
}

// 5-point anisotropic Poisson on a side x side grid, Dirichlet boundary
// (config 5): index r*side + c; neighbours (r,c±1) weigh ax, (r±1,c) ay.
int pmmf_b200_workload_aniso_grid(int64_t side, double ax, double ay, pmmf_b200_workload* out) {
  if (side < 1) return 1;
  const int64_t n = side * side;
  Coo coo;
  coo.r.reserve(5 * n);
  coo.c.reserve(5 * n);
  coo.v.reserve(5 * n);
  const double diag = 2.0 * ax + 2.0 * ay;
  for (int64_t r = 0; r < side; ++r)
    for (int64_t c = 0; c < side; ++c) {
      const int64_t i = r * side + c;
      if (r > 0) coo.push(i, i - side, -ay);
      if (c > 0) coo.push(i, i - 1, -ax);
      coo.push(i, i, diag);
      if (c + 1 < side) coo.push(i, i + 1, -ax);
      if (r + 1 < side) coo.push(i, i + side, -ay);
    }
  return emit(coo, n, out);
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
