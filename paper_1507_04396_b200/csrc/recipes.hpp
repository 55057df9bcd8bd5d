// recipes.hpp — the seeded input recipes of SURVEY.md §8(d), written once
// over any random source with the reference's draw interface
// (uniform01(), normal(): rng.hpp:53-71).
//
// workloads.cpp instantiates them on the library's own generator
// (pmmf_b200::Xoshiro, rng.cuh); oracle/ref_driver.cpp instantiates them on
// the reference's pmmf::Rng, so the CPU reference arm of bench.py builds its
// input without loading libpmmf_b200.so, and tests/test_workloads.py checks
// that both instantiations emit identical triplets.
//
// The reference ships no R-MAT / RBF / anisotropic generators (SURVEY.md
// Appendix B, graphs.hpp).  Output is COO in emission order.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

namespace pmmf_recipes {

struct Coo {
  int64_t n = 0;
  std::vector<int64_t> r, c;
  std::vector<double> v;
  void push(int64_t i, int64_t j, double x) {
    r.push_back(i);
    c.push_back(j);
    v.push_back(x);
  }
  void reserve(std::size_t m) {
    r.reserve(m);
    c.reserve(m);
    v.reserve(m);
  }
};

// R-MAT graph (a,b,c,d = .57,.19,.19,.05), (epv·n)/2 edge samples, self
// loops dropped, deduplicated; normalized Laplacian + shift·I.
template <class Rng>
bool rmat(int32_t scale, int32_t edges_per_vertex, Rng& rng, double shift, Coo& coo) {
  if (scale < 1 || scale > 30 || edges_per_vertex < 1) return false;
  const int64_t n = int64_t{1} << scale;
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
  coo.n = n;
  coo.reserve(2 * edges.size() + static_cast<std::size_t>(n));
  for (uint64_t e : edges) {
    const int64_t i = static_cast<int64_t>(e >> 32), j = static_cast<int64_t>(e & 0xffffffffull);
    const double w = -1.0 / std::sqrt(static_cast<double>(deg[i]) * static_cast<double>(deg[j]));
    coo.push(i, j, w);
    coo.push(j, i, w);
  }
  for (int64_t i = 0; i < n; ++i) coo.push(i, i, (deg[i] > 0 ? 1.0 : 0.0) + shift);
  return true;
}

// Dense SPD A = X X^T / d + shift·I, X n x d ~ N(0,1) row-major (config 1).
template <class Rng>
bool dense_spd(int64_t n, int64_t d, Rng& rng, double shift, Coo& coo) {
  if (n < 1 || d < 1) return false;
  std::vector<double> x(static_cast<std::size_t>(n * d));
  for (auto& v : x) v = rng.normal();
  coo.n = n;
  coo.reserve(static_cast<std::size_t>(n * n));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double s = 0.0;
      for (int64_t t = 0; t < d; ++t) s += x[i * d + t] * x[j * d + t];
      s /= static_cast<double>(d);
      if (i == j) s += shift;
      coo.push(i, j, s);
    }
  return true;
}

// Gaussian RBF kernel on n uniform points in [0,1]^dim (config 3):
// K_ij = exp(-|x_i - x_j|^2 / (2 bw^2)) + shift·delta_ij.
template <class Rng>
bool rbf(int64_t n, int32_t dim, double bandwidth, Rng& rng, double shift, Coo& coo) {
  if (n < 1 || dim < 1) return false;
  std::vector<double> x(static_cast<std::size_t>(n * dim));
  for (auto& v : x) v = rng.uniform01();
  const double denom = 2.0 * bandwidth * bandwidth;
  coo.n = n;
  coo.reserve(static_cast<std::size_t>(n * n));
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
  return true;
}

// 5-point anisotropic Poisson on a side x side grid, Dirichlet boundary
// (config 5): index r*side + c; neighbours (r,c±1) weigh ax, (r±1,c) ay.
inline bool aniso_grid(int64_t side, double ax, double ay, Coo& coo) {
  if (side < 1) return false;
  const int64_t n = side * side;
  coo.n = n;
  coo.reserve(static_cast<std::size_t>(5 * n));
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
  return true;
}

}  // namespace pmmf_recipes
