// rotation.cuh — k x k rotation arithmetic, bit-exact with the reference,
// usable from the search kernel's scalar lane and from the host C-ABI.
//   jacobi_angle        dense.hpp:132-138
//   jacobi_diagonalize  dense.hpp:144-183 (cyclic, rel_tol 1e-15, 64 sweeps)
//   rotation_from_gram  factorizer.hpp:150-171 (+ fix_row_signs :130-144)
//   corner conjugation  sparse.hpp:403 via DenseMatrix::multiply (dense.hpp:55-65)
// Compiled with -fmad=false: every product and sum rounds separately.
#pragma once

#include <cmath>

#ifdef __CUDACC__
#define PMMF_HDI __host__ __device__ inline
#else
#define PMMF_HDI inline
#endif

namespace pmmf_b200 {

constexpr int kMaxK = 8;

PMMF_HDI void jacobi_angle(double gpp, double grr, double gpr, double& c, double& s) {
  if (gpr == 0.0) {
    c = 1.0;
    s = 0.0;
    return;
  }
  const double tau = (grr - gpp) / (2.0 * gpr);
  const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
  c = 1.0 / sqrt(1.0 + t * t);
  s = t * c;
}

// Loop policies for the cyclic Jacobi below.  SeqLoop: the calling thread
// runs every loop (the search kernel's scalar lane, the host).  CtaLoop (see
// operator.cu): the per-pair row / column updates are independent over t and
// run strided over a CTA, with barriers between dependent steps; sums whose
// order matters run on the leader thread and are broadcast.  Every matrix
// element sees the same operation sequence under both policies.
struct SeqLoop {
  template <class F>
  PMMF_HDI void each(int n, F&& f) const {
    for (int t = 0; t < n; ++t) f(t);
  }
  PMMF_HDI void sync() const {}
  PMMF_HDI bool leader() const { return true; }
  PMMF_HDI double bcast(double v) const { return v; }
};

// Cyclic Jacobi (jacobi_diagonalize, dense.hpp:144-183; rel_tol 1e-15, 64
// sweeps) on accessors a(i, j), q(i, j): a is diagonalized in place, q
// receives the rotation (q a q^T diagonal).
template <class MA, class MQ, class Par>
PMMF_HDI void jacobi_diagonalize_g(MA a, MQ q, int n, const Par& par) {
  par.each(n * n, [&](int x) { q(x / n, x % n) = (x / n == x % n) ? 1.0 : 0.0; });
  double fro = 0.0;
  if (par.leader())
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) fro += a(i, j) * a(i, j);
  const double scale = sqrt(par.bcast(fro));
  if (scale == 0.0 || n < 2) return;
  const double stop = 1e-15 * scale;
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = 0.0;
    if (par.leader())
      for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) off += 2.0 * a(i, j) * a(i, j);
    if (sqrt(par.bcast(off)) <= stop) break;
    for (int p = 0; p < n; ++p)
      for (int r = p + 1; r < n; ++r) {
        const double apr = a(p, r);
        if (apr == 0.0) continue;
        double c, s;
        jacobi_angle(a(p, p), a(r, r), apr, c, s);
        par.sync();  // every thread has read the pivot entries
        par.each(n, [&](int t) {
          const double ap = a(p, t), ar = a(r, t);
          a(p, t) = c * ap - s * ar;
          a(r, t) = s * ap + c * ar;
        });
        par.sync();
        par.each(n, [&](int t) {
          const double ap = a(t, p), ar = a(t, r);
          a(t, p) = c * ap - s * ar;
          a(t, r) = s * ap + c * ar;
          const double qp = q(p, t), qr = q(r, t);
          q(p, t) = c * qp - s * qr;
          q(r, t) = s * qp + c * qr;
        });
        par.sync();
        if (par.leader()) {
          a(p, r) = 0.0;
          a(r, p) = 0.0;
        }
        par.sync();
      }
  }
}

// Row-major view with a fixed stride.
struct RowMajor {
  double* p;
  int ld;
  PMMF_HDI double& operator()(int i, int j) const { return p[static_cast<long long>(i) * ld + j]; }
};

// a (n x n, row-major stride kMaxK) is diagonalized in place; q returned.
PMMF_HDI void jacobi_diagonalize(double (*a)[kMaxK], int n, double (*q)[kMaxK]) {
  jacobi_diagonalize_g(RowMajor{&a[0][0], kMaxK}, RowMajor{&q[0][0], kMaxK}, n, SeqLoop{});
}

// Returns false when g is not symmetric within 1e-9 * max(1, max|g|)
// (the reference throws std::invalid_argument there).
PMMF_HDI bool rotation_from_gram(const double (*g)[kMaxK], int k, double (*q)[kMaxK]) {
  double asym = 0.0, mx = 0.0;
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) {
      mx = fmax(mx, fabs(g[i][j]));
      if (j > i) asym = fmax(asym, fabs(g[i][j] - g[j][i]));
    }
  if (asym > 1e-9 * fmax(1.0, mx)) return false;
  double w[kMaxK][kMaxK];
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) w[i][j] = 0.5 * (g[i][j] + g[j][i]);
  if (k == 2) {
    double c, s;
    jacobi_angle(w[0][0], w[1][1], w[0][1], c, s);
    q[0][0] = c;
    q[0][1] = -s;
    q[1][0] = s;
    q[1][1] = c;
  } else {
    jacobi_diagonalize(w, k, q);
  }
  for (int i = 0; i < k; ++i) {
    int arg = 0;
    double best = fabs(q[i][0]);
    for (int j = 1; j < k; ++j)
      if (fabs(q[i][j]) > best) {
        best = fabs(q[i][j]);
        arg = j;
      }
    if (q[i][arg] < 0.0)
      for (int j = 0; j < k; ++j) q[i][j] = -q[i][j];
  }
  return true;
}

// out = (q * C) * q^T with DenseMatrix::multiply's loop order and its
// zero-left-factor skip.
PMMF_HDI void conjugate_corner(const double (*q)[kMaxK], const double (*C)[kMaxK], int k, double (*out)[kMaxK]) {
  double p[kMaxK][kMaxK];
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) p[i][j] = 0.0;
  for (int i = 0; i < k; ++i)
    for (int t = 0; t < k; ++t) {
      const double x = q[i][t];
      if (x == 0.0) continue;
      for (int j = 0; j < k; ++j) p[i][j] += x * C[t][j];
    }
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) out[i][j] = 0.0;
  for (int i = 0; i < k; ++i)
    for (int t = 0; t < k; ++t) {
      const double x = p[i][t];
      if (x == 0.0) continue;
      for (int j = 0; j < k; ++j) out[i][j] += x * q[j][t];  // q^T(t, j) = q(j, t)
    }
}

PMMF_HDI bool is_exact_identity(const double (*q)[kMaxK], int k) {
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j)
      if (q[i][j] != (i == j ? 1.0 : 0.0)) return false;
  return true;
}

// off_diag_norm_sq (factorizer.hpp:122-124) with std::max's NaN behaviour.
PMMF_HDI double off_diag_norm_sq(double ns, double d) {
  const double x = ns - d * d;
  return (0.0 < x) ? x : 0.0;
}

}  // namespace pmmf_b200

namespace pmmf_b200 {

// ---- compile-time-K variants (register resident in device code) --------
template <int K>
PMMF_HDI bool rotation_from_gram_k(const double (&g)[K][K], double (&q)[K][K]) {
  double gg[kMaxK][kMaxK], qq[kMaxK][kMaxK];
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) gg[i][j] = g[i][j];
  const bool ok = rotation_from_gram(gg, K, qq);
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) q[i][j] = qq[i][j];
  return ok;
}

template <>
PMMF_HDI bool rotation_from_gram_k<2>(const double (&g)[2][2], double (&q)[2][2]) {
  const double asym = fabs(g[0][1] - g[1][0]);
  const double mx = fmax(fmax(fabs(g[0][0]), fabs(g[0][1])), fmax(fabs(g[1][0]), fabs(g[1][1])));
  if (asym > 1e-9 * fmax(1.0, mx)) return false;
  const double w00 = 0.5 * (g[0][0] + g[0][0]);
  const double w11 = 0.5 * (g[1][1] + g[1][1]);
  const double w01 = 0.5 * (g[0][1] + g[1][0]);
  double c, s;
  jacobi_angle(w00, w11, w01, c, s);
  q[0][0] = c;
  q[0][1] = -s;
  q[1][0] = s;
  q[1][1] = c;
  // fix_row_signs (factorizer.hpp:130-144)
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int arg = fabs(q[i][1]) > fabs(q[i][0]) ? 1 : 0;
    if (q[i][arg] < 0.0) {
      q[i][0] = -q[i][0];
      q[i][1] = -q[i][1];
    }
  }
  return true;
}

template <int K>
PMMF_HDI void conjugate_corner_k(const double (&q)[K][K], const double (&C)[K][K], double (&out)[K][K]) {
  double p[K][K];
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) p[i][j] = 0.0;
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int t = 0; t < K; ++t) {
      const double x = q[i][t];
      if (x != 0.0) {
#pragma unroll
        for (int j = 0; j < K; ++j) p[i][j] += x * C[t][j];
      }
    }
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) out[i][j] = 0.0;
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int t = 0; t < K; ++t) {
      const double x = p[i][t];
      if (x != 0.0) {
#pragma unroll
        for (int j = 0; j < K; ++j) out[i][j] += x * q[j][t];
      }
    }
}

template <int K>
PMMF_HDI bool is_exact_identity_k(const double (&q)[K][K]) {
  bool id = true;
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) id = id && q[i][j] == (i == j ? 1.0 : 0.0);
  return id;
}

}  // namespace pmmf_b200
