// precond.cu — the comparison preconditioners of the CG study
// (solver.hpp:222-340: Jacobi, SSOR, IC(0)) and the uniform Nystrom sketch
// (transform_ops.hpp:252-307) on the device.
//
// Data: the lower triangle of A in global ids (extract_lower,
// solver.hpp:204-218) as a CSC (column j -> rows r > j ascending) plus a
// CSR view of the same entries (row r -> columns j < r ascending, with the
// entry's CSC position), the diagonal separately.  Stored zeros are kept, as
// the reference's blocked storage keeps them (sparse.hpp:66-79): they belong
// to the IC(0) pattern.
//
// Triangular solves and the IC(0) factorization are "sync-free": warps take
// rows (columns) in dependency order from an atomic ticket, spin on the
// ready flags of the rows they read, compute, and publish their own flag.
// A row is only ever waited on after its ticket was taken by a running warp,
// so the lowest unfinished row always makes progress (no deadlock for any
// grid size).  Each row's arithmetic is the reference's sequential order:
//   forward_solve (solver.hpp:183-191): x_r = (b_r - sum_{j<r, ascending}
//     L_rj x_j) / d_r — the column-oriented loop subtracts from x_r in
//     ascending j, so a row-oriented accumulation is the same sequence;
//   backward_solve (:193-201): column j of L read as row j of L^T;
//   IC(0) (:278-313): left-looking column j, pivot and the entries below it
//     updated for every k of row j in ascending k (rows[j] is filled in
//     column order).
// The critical path is the dependency depth (2n^(1/2) levels on a 2-D
// grid), one L2 round trip per level.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "engine.cuh"
#include "layout.cuh"
#include "precond.cuh"
#include "rng.cuh"

namespace pmmf_b200 {

int guarded_call(char* err, size_t errlen, void (*fn)(void*), void* ctx);

namespace {

template <typename F>
int guarded(char* err, size_t errlen, F&& f) {
  return guarded_call(err, errlen, [](void* c) { (*static_cast<F*>(c))(); }, &f);
}

constexpr int kThreads = 256;

__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ int ld_flag(const int* p) { return *reinterpret_cast<const volatile int*>(p); }

// ------------------------------------------------------------ extraction
// One pass over the stored entries (stage CSC): the diagonal by global id,
// strictly lower entries appended with a (col, row) key (appending order is
// irrelevant: keys are unique and sorted next).
__global__ void k_split_lower(i64 N, const i64* __restrict__ ptr, const int32_t* __restrict__ row,
                              const double* __restrict__ val, const int32_t* __restrict__ s2g, i64 n,
                              double* __restrict__ diag, uint8_t* __restrict__ has_diag,
                              unsigned long long* __restrict__ cnt, uint64_t* __restrict__ key,
                              double* __restrict__ kval) {
  const i64 c = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (c >= N) return;
  const i64 gc = s2g[c];
  for (i64 e = ptr[c]; e < ptr[c + 1]; ++e) {
    const i64 gr = s2g[row[e]];
    if (gr == gc) {
      diag[gr] = val[e];
      has_diag[gr] = 1;
    } else if (gr > gc) {
      const unsigned long long o = atomicAdd(cnt, 1ull);
      key[o] = static_cast<uint64_t>(gc) * static_cast<uint64_t>(n) + static_cast<uint64_t>(gr);
      kval[o] = val[e];
    }
  }
}

// ptr[c] = first position whose major index is >= c (sorted majors).
__global__ void k_ptr_from_sorted(i64 m, const uint64_t* __restrict__ key, uint64_t n, bool major_is_quot, i64 nmaj,
                                  i64* __restrict__ ptr) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i > m) return;
  auto major = [&](i64 p) -> i64 {
    return major_is_quot ? static_cast<i64>(key[p] / n) : static_cast<i64>(key[p] % n);
  };
  const i64 cur = i < m ? major(i) : nmaj;
  const i64 prev = i > 0 ? major(i - 1) : -1;
  for (i64 c = prev + 1; c <= cur; ++c) ptr[c] = i;
}

__global__ void k_unpack_csc(i64 m, const uint64_t* __restrict__ key, uint64_t n, int32_t* __restrict__ crow) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < m) crow[i] = static_cast<int32_t>(key[i] % n);
}

// Row-major keys (row, col) of the CSC entries, payload = CSC position.
__global__ void k_row_keys(i64 m, const uint64_t* __restrict__ ckey, uint64_t n, uint64_t* __restrict__ rkey,
                           i64* __restrict__ pos) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= m) return;
  const uint64_t col = ckey[i] / n, row = ckey[i] % n;
  rkey[i] = row * n + col;
  pos[i] = i;
}

__global__ void k_unpack_csr(i64 m, const uint64_t* __restrict__ rkey, uint64_t n, int32_t* __restrict__ rcol) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < m) rcol[i] = static_cast<int32_t>(rkey[i] % n);
}

// Row sums of |a_ij| in the reference's to_triplets order (columns by stage
// id, blocked_matrix.hpp:422-436) and the compensation ratio
// (solver.hpp:318-327): first non-positive diagonal by global id, max ratio.
__global__ void k_ic_ratio(i64 N, const i64* __restrict__ tptr, const int32_t* __restrict__ tcol,
                           const double* __restrict__ tval, const int32_t* __restrict__ s2g,
                           const double* __restrict__ diag, unsigned long long* __restrict__ first_bad,
                           unsigned long long* __restrict__ max_bits) {
  const i64 r = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (r >= N) return;
  const i64 g = s2g[r];
  double sum = 0.0;
  for (i64 e = tptr[r]; e < tptr[r + 1]; ++e) sum = dadd(sum, fabs(tval[e]));
  const double d = diag[g];
  if (!(d > 0.0)) {
    atomicMin(first_bad, static_cast<unsigned long long>(g));
    return;
  }
  const double ratio = ddiv(sum, d);
  atomicMax(max_bits, static_cast<unsigned long long>(__double_as_longlong(ratio)));
}

__global__ void k_first_zero(i64 n, const double* __restrict__ diag, unsigned long long* __restrict__ first) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < n && diag[i] == 0.0) atomicMin(first, static_cast<unsigned long long>(i));
}

// ------------------------------------------------------------ elementwise
__global__ void k_jacobi_scale(i64 n, const double* __restrict__ diag, const uint8_t* __restrict__ has,
                               double* __restrict__ scale) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double d = diag[i];
  scale[i] = (has[i] && d > 0.0) ? ddiv(1.0, sqrt(d)) : 0.0;
}

// SSOR setup (solver.hpp:243-250): sqrt_d = front * sqrt(|d|), d <- d / omega.
__global__ void k_ssor_setup(i64 n, double front, double omega, double* __restrict__ diag,
                             double* __restrict__ sqrt_d) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double d = diag[i];
  sqrt_d[i] = dmul(front, sqrt(fabs(d)));
  diag[i] = ddiv(d, omega);
}

__global__ void k_boost(i64 n, const double* __restrict__ d0, double f, double* __restrict__ d) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < n) d[i] = dmul(d0[i], f);
}

// out[i, r] = s[i] * in[i, r]
__global__ void k_scale_rows(i64 n, int nr, const double* __restrict__ s, const double* __restrict__ in,
                             double* __restrict__ out) {
  const i64 x = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (x >= n * nr) return;
  out[x] = dmul(s[x / nr], in[x]);
}
// v[i, r] *= s[i]  (forward_solve's result scaled in place, solver.hpp:252-255)
__global__ void k_scale_rows_inplace(i64 n, int nr, const double* __restrict__ s, double* __restrict__ v) {
  const i64 x = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (x >= n * nr) return;
  v[x] = dmul(v[x], s[x / nr]);
}

// ------------------------------------------------------------ sync-free solves
// kBack = false: x = (D + L)^-1 b with (ptr, idx, val) the CSR view of L
// (row j -> columns < j); kBack = true: x = (D + L)^-T b with the CSC of L
// (column j -> rows > j), rows handed out from n-1 down.  val_pos maps the
// CSR view onto the CSC value array (nullptr: val is indexed directly).
template <bool kBack>
__global__ void __launch_bounds__(kThreads) k_trsv(i64 n, int nr, const i64* __restrict__ ptr,
                                                   const int32_t* __restrict__ idx, const i64* __restrict__ val_pos,
                                                   const double* __restrict__ val, const double* __restrict__ diag,
                                                   const double* __restrict__ b, double* x, int* flag, int epoch,
                                                   unsigned long long* ticket) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= static_cast<unsigned long long>(n)) return;
    const i64 j = kBack ? n - 1 - static_cast<i64>(t) : static_cast<i64>(t);
    const i64 e0 = ptr[j], e1 = ptr[j + 1];
    for (i64 e = e0 + lane; e < e1; e += 32)
      while (ld_flag(flag + idx[e]) != epoch) {
      }
    __threadfence();
    __syncwarp();
    const double dj = diag[j];
    for (int r = lane; r < nr; r += 32) {
      double acc = b[j * nr + r];
      for (i64 e = e0; e < e1; ++e) {
        const double v = val_pos ? val[val_pos[e]] : val[e];
        acc = dsub(acc, dmul(v, __ldcg(x + static_cast<i64>(idx[e]) * nr + r)));
      }
      __stcg(x + j * nr + r, ddiv(acc, dj));
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicExch(flag + j, epoch);
  }
}

// IC(0), left-looking (solver.hpp:284-313).  cval holds A's lower values on
// entry and L's on exit; diag holds the boosted diagonal on entry and
// sqrt(pivot) on exit.  A breakdown (!(pivot > 0)) is flagged; the column
// still publishes (NaNs) so no waiter blocks.
__global__ void __launch_bounds__(kThreads) k_ic0(i64 n, const i64* __restrict__ cptr,
                                                  const int32_t* __restrict__ crow, double* cval, double* diag,
                                                  const i64* __restrict__ rptr, const int32_t* __restrict__ rcol,
                                                  const i64* __restrict__ rpos, int* flag, int epoch,
                                                  unsigned long long* ticket, int* broke) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= static_cast<unsigned long long>(n)) return;
    const i64 j = static_cast<i64>(t);
    const i64 c0 = cptr[j];
    const int len = static_cast<int>(cptr[j + 1] - c0);
    double pivot = diag[j];
    for (i64 e = rptr[j]; e < rptr[j + 1]; ++e) {
      const int k = rcol[e];
      const i64 p = rpos[e];
      if (lane == 0)
        while (ld_flag(flag + k) != epoch) {
        }
      __syncwarp();
      __threadfence();
      const double ljk = __ldcg(cval + p);
      pivot = dsub(pivot, dmul(ljk, ljk));
      const i64 k1 = cptr[k + 1];
      for (i64 s = p + 1 + lane; s < k1; s += 32) {
        const int r = crow[s];
        int lo = 0, hi = len;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (crow[c0 + mid] < r) lo = mid + 1; else hi = mid;
        }
        if (lo < len && crow[c0 + lo] == r) __stcg(cval + c0 + lo, dsub(__ldcg(cval + c0 + lo), dmul(__ldcg(cval + s), ljk)));
      }
      __syncwarp();
    }
    if (!(pivot > 0.0) && lane == 0) atomicExch(broke, 1);
    const double d = sqrt(pivot);
    for (int q = lane; q < len; q += 32) __stcg(cval + c0 + q, ddiv(__ldcg(cval + c0 + q), d));
    if (lane == 0) __stcg(diag + j, d);
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicExch(flag + j, epoch);
  }
}

int sync_free_grid(i64 n) {
  static const int cap = [] {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) (void)cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    (void)cudaGetLastError();
    return sms * (2048 / kThreads);
  }();
  return static_cast<int>(std::max<i64>(1, std::min<i64>(cap, (n + 7) / 8)));
}

template <typename K, typename V>
void radix_sort_pairs(DBuf<K>& keys, DBuf<V>& vals, i64 m, int end_bit, cudaStream_t s) {
  if (m <= 1) return;
  DBuf<K> k2(m, s);
  DBuf<V> v2(m, s);
  cub::DoubleBuffer<K> kb(keys.get(), k2.get());
  cub::DoubleBuffer<V> vb(vals.get(), v2.get());
  size_t tmp = 0;
  PMMF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, static_cast<int64_t>(m), 0, end_bit, s));
  DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
  PMMF_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, kb, vb, static_cast<int64_t>(m), 0, end_bit, s));
  if (kb.Current() != keys.get()) {
    std::swap(keys, k2);
    std::swap(vals, v2);
  }
}

// ------------------------------------------------------------ the matrix
// from_triplets (with the input partition, blocked_matrix.hpp:138-156,
// stored zeros kept) followed by extract_lower, all on the device.
struct Lower {
  i64 n = 0, m = 0;  // dimension, strictly lower entries
  DBuf<double> diag;
  DBuf<uint8_t> has_diag;
  DBuf<i64> cptr, rptr, rpos;
  DBuf<int32_t> crow, rcol;
  DBuf<double> cval;
  // transpose of the stage CSC (rows with columns in stage order) for the
  // IC compensation's row sums
  Csc T;
  Numbering nb;
};

struct Stream {
  cudaStream_t s = nullptr;
  Stream() { PMMF_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~Stream() {
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
};

void build_lower(Lower& L, const pmmf_b200_coo* a, bool need_rows, cudaStream_t s) {
  const i64 n = a->n;
  L.n = n;
  {
    std::vector<std::vector<i64>> init;
    if (a->n_clusters == 0) {
      init.emplace_back(static_cast<size_t>(std::max<i64>(n, 0)));
      std::iota(init[0].begin(), init[0].end(), i64{0});
    } else {
      for (i64 u = 0; u < a->n_clusters; ++u)
        init.emplace_back(a->cluster_members + a->cluster_offsets[u], a->cluster_members + a->cluster_offsets[u + 1]);
    }
    L.nb.build(init, std::max<i64>(n, 0), s);
  }
  Csc A;
  {
    const int64_t* rows = a->rows;
    const int64_t* cols = a->cols;
    const double* vals = a->vals;
    DBuf<int64_t> dr, dc;
    DBuf<double> dv;
    if (!a->on_device && a->nnz > 0) {
      dr.alloc(a->nnz, s);
      dc.alloc(a->nnz, s);
      dv.alloc(a->nnz, s);
      dr.upload(a->rows, a->nnz);
      dc.upload(a->cols, a->nnz);
      dv.upload(a->vals, a->nnz);
      rows = dr.get();
      cols = dc.get();
      vals = dv.get();
    }
    csc_from_coo(A, L.nb, n, a->nnz, rows, cols, vals, s, /*keep_zeros=*/true);
  }
  const i64 N = A.N;
  L.diag.alloc(std::max<i64>(n, 1), s);
  L.diag.zero();
  L.has_diag.alloc(std::max<i64>(n, 1), s);
  L.has_diag.zero();
  DBuf<unsigned long long> cnt(1, s);
  cnt.zero();
  DBuf<uint64_t> key(std::max<i64>(A.nnz, 1), s);
  DBuf<double> kval(std::max<i64>(A.nnz, 1), s);
  PMMF_LAUNCH(k_split_lower, blocks_for(N, kThreads), kThreads, 0, s, N, A.ptr.get(), A.row.get(), A.val.get(),
              L.nb.d_s2g.get(), n, L.diag.get(), L.has_diag.get(), cnt.get(), key.get(), kval.get());
  const i64 m = static_cast<i64>(cnt.to_host(1)[0]);
  L.m = m;
  const uint64_t un = static_cast<uint64_t>(std::max<i64>(n, 1));
  const int kb = std::max(1, bits_for(std::max<i64>(n, 1) * std::max<i64>(n, 1) - 1));
  radix_sort_pairs(key, kval, m, kb, s);
  L.cval = std::move(kval);
  L.crow.alloc(std::max<i64>(m, 1), s);
  L.cptr.alloc(n + 1, s);
  PMMF_LAUNCH(k_unpack_csc, blocks_for(m, kThreads), kThreads, 0, s, m, key.get(), un, L.crow.get());
  PMMF_LAUNCH(k_ptr_from_sorted, blocks_for(m + 1, kThreads), kThreads, 0, s, m, key.get(), un, true, n,
              L.cptr.get());
  if (need_rows) {
    DBuf<uint64_t> rkey(std::max<i64>(m, 1), s);
    L.rpos.alloc(std::max<i64>(m, 1), s);
    PMMF_LAUNCH(k_row_keys, blocks_for(m, kThreads), kThreads, 0, s, m, key.get(), un, rkey.get(), L.rpos.get());
    radix_sort_pairs(rkey, L.rpos, m, kb, s);
    L.rcol.alloc(std::max<i64>(m, 1), s);
    L.rptr.alloc(n + 1, s);
    PMMF_LAUNCH(k_unpack_csr, blocks_for(m, kThreads), kThreads, 0, s, m, rkey.get(), un, L.rcol.get());
    PMMF_LAUNCH(k_ptr_from_sorted, blocks_for(m + 1, kThreads), kThreads, 0, s, m, rkey.get(), un, true, n,
                L.rptr.get());
  }
  Paged P;
  paged_from_csc(P, std::move(A), 1, s);
  transpose_paged(L.T, P, s);
  PMMF_CUDA(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------ preconditioners
struct DevPrecond : SplitPrecond {
  DBuf<int> flag;
  DBuf<unsigned long long> ticket;
  int epoch = 0;
  void init_sync(i64 nn, cudaStream_t s) {
    flag.alloc(std::max<i64>(nn, 1), s);
    flag.zero();
    ticket.alloc(1, s);
  }
  int next_epoch() {
    if (++epoch == 0x7fffffff) epoch = 1;  // flags are compared for equality only
    return epoch;
  }
  void solve(bool back, const Lower& L, const double* diag, int nr, const double* b, double* x, cudaStream_t s) {
    if (L.n == 0) return;
    // on the caller's stream: the ticket is reset in order with the solve
    PMMF_CUDA(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned long long), s));
    const int ep = next_epoch();
    if (!back)
      PMMF_LAUNCH(k_trsv<false>, sync_free_grid(L.n), kThreads, 0, s, L.n, nr, L.rptr.get(), L.rcol.get(),
                  L.rpos.get(), L.cval.get(), diag, b, x, flag.get(), ep, ticket.get());
    else
      PMMF_LAUNCH(k_trsv<true>, sync_free_grid(L.n), kThreads, 0, s, L.n, nr, L.cptr.get(), L.crow.get(),
                  static_cast<const i64*>(nullptr), L.cval.get(), diag, b, x, flag.get(), ep, ticket.get());
  }
};

struct JacobiPre : DevPrecond {
  DBuf<double> scale;
  void apply(int, int nr, const double* in, double* out, cudaStream_t s) override {
    PMMF_LAUNCH(k_scale_rows, blocks_for(n * nr, kThreads), kThreads, 0, s, n, nr, scale.get(), in, out);
  }
};

struct SsorPre : DevPrecond {
  Lower L;
  DBuf<double> sqrt_d;
  DBuf<double> tmp;
  void apply(int side, int nr, const double* in, double* out, cudaStream_t s) override {
    if (side == 0) {  // K^-1 = sqrt_d .* forward_solve
      solve(false, L, L.diag.get(), nr, in, out, s);
      PMMF_LAUNCH(k_scale_rows_inplace, blocks_for(n * nr, kThreads), kThreads, 0, s, n, nr, sqrt_d.get(), out);
    } else {  // K^-T = backward_solve(sqrt_d .* in)
      if (tmp.n < n * nr) {  // grown on the handle's stream, ordered before use
        tmp.alloc(n * nr, own);
        PMMF_CUDA(cudaStreamSynchronize(own));
      }
      PMMF_LAUNCH(k_scale_rows, blocks_for(n * nr, kThreads), kThreads, 0, s, n, nr, sqrt_d.get(), in, tmp.get());
      solve(true, L, L.diag.get(), nr, tmp.get(), out, s);
    }
  }
};

struct IcPre : DevPrecond {
  Lower L;
  void apply(int side, int nr, const double* in, double* out, cudaStream_t s) override {
    solve(side != 0, L, L.diag.get(), nr, in, out, s);
  }
};

std::string num(i64 v) { return std::to_string(v); }

}  // namespace

std::unique_ptr<SplitPrecond> make_precond(const pmmf_b200_coo* a, int kind, double omega) {
  if (!a) fail(PMMF_INVALID_ARGUMENT, "preconditioner: null matrix");
  if (kind == PMMF_PRECOND_SSOR && !(omega > 0.0 && omega < 2.0))
    fail(PMMF_INVALID_ARGUMENT, "ssor: omega must be in (0, 2)");
  if (kind != PMMF_PRECOND_JACOBI && kind != PMMF_PRECOND_SSOR && kind != PMMF_PRECOND_IC)
    fail(PMMF_INVALID_ARGUMENT, "preconditioner: unknown kind");
  PMMF_CUDA(cudaSetDevice(a->device));
  const i64 n = a->n;
  if (kind == PMMF_PRECOND_JACOBI) {
    auto p = std::make_unique<JacobiPre>();
    cudaStream_t s = p->own;
    p->kind = kind;
    p->n = n;
    p->device = a->device;
    Lower L;
    build_lower(L, a, false, s);
    p->scale.alloc(std::max<i64>(n, 1), s);
    PMMF_LAUNCH(k_jacobi_scale, blocks_for(n, kThreads), kThreads, 0, s, n, L.diag.get(), L.has_diag.get(),
                p->scale.get());
    PMMF_CUDA(cudaStreamSynchronize(s));
    return p;
  }
  if (kind == PMMF_PRECOND_SSOR) {
    auto p = std::make_unique<SsorPre>();
    cudaStream_t s = p->own;
    p->kind = kind;
    p->n = n;
    p->device = a->device;
    build_lower(p->L, a, true, s);
    DBuf<unsigned long long> first(1, s);
    first.fill_bytes(0xff);
    PMMF_LAUNCH(k_first_zero, blocks_for(n, kThreads), kThreads, 0, s, n, p->L.diag.get(), first.get());
    const unsigned long long f = first.to_host(1)[0];
    if (f != ~0ull) fail(PMMF_NUMERIC, "ssor: zero diagonal entry at row " + num(static_cast<i64>(f)));
    const double front = std::sqrt((2.0 - omega) / omega);
    p->sqrt_d.alloc(std::max<i64>(n, 1), s);
    PMMF_LAUNCH(k_ssor_setup, blocks_for(n, kThreads), kThreads, 0, s, n, front, omega, p->L.diag.get(),
                p->sqrt_d.get());
    p->init_sync(n, s);
    PMMF_CUDA(cudaStreamSynchronize(s));
    return p;
  }
  // IC(0) with one compensated restart (solver.hpp:315-333)
  auto p = std::make_unique<IcPre>();
  cudaStream_t s = p->own;
  p->kind = kind;
  p->n = n;
  p->device = a->device;
  Lower& L = p->L;
  build_lower(L, a, true, s);
  p->init_sync(n, s);
  DBuf<double> a_val(std::max<i64>(L.m, 1), s), a_diag(std::max<i64>(n, 1), s);
  if (L.m) PMMF_CUDA(cudaMemcpyAsync(a_val.get(), L.cval.get(), sizeof(double) * L.m, cudaMemcpyDeviceToDevice, s));
  if (n) PMMF_CUDA(cudaMemcpyAsync(a_diag.get(), L.diag.get(), sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  DBuf<int> broke(1, s);
  auto attempt = [&](double boost) -> bool {
    if (L.m) PMMF_CUDA(cudaMemcpyAsync(L.cval.get(), a_val.get(), sizeof(double) * L.m, cudaMemcpyDeviceToDevice, s));
    PMMF_LAUNCH(k_boost, blocks_for(n, kThreads), kThreads, 0, s, n, a_diag.get(), 1.0 + boost, L.diag.get());
    broke.zero();
    p->ticket.zero();
    const int ep = p->next_epoch();
    PMMF_LAUNCH(k_ic0, sync_free_grid(n), kThreads, 0, s, n, L.cptr.get(), L.crow.get(), L.cval.get(), L.diag.get(),
                L.rptr.get(), L.rcol.get(), L.rpos.get(), p->flag.get(), ep, p->ticket.get(), broke.get());
    return broke.to_host(1)[0] == 0;
  };
  if (!attempt(0.0)) {
    DBuf<unsigned long long> first(1, s), mx(1, s);
    first.fill_bytes(0xff);
    mx.zero();
    PMMF_LAUNCH(k_ic_ratio, blocks_for(L.T.N, kThreads), kThreads, 0, s, L.T.N, L.T.ptr.get(), L.T.row.get(),
                L.T.val.get(), L.nb.d_s2g.get(), a_diag.get(), first.get(), mx.get());
    const unsigned long long f = first.to_host(1)[0];
    if (f != ~0ull)
      fail(PMMF_NUMERIC, "ic: non-positive diagonal, cannot compensate row " + num(static_cast<i64>(f)));
    const unsigned long long bits = mx.to_host(1)[0];
    double alpha = 0.0;
    std::memcpy(&alpha, &bits, sizeof(alpha));
    p->compensated = 1;
    p->alpha = alpha;
    if (!attempt(alpha)) fail(PMMF_NUMERIC, "ic: breakdown persists after diagonal compensation");
  }
  PMMF_CUDA(cudaStreamSynchronize(s));
  return p;
}

// ================================================================ Nystrom
namespace {

// Row-major dense n x n from the stage CSC (dense_from_blocked,
// transform_ops.hpp:215-220; entries unique after from_triplets).
__global__ void k_dense_from_csc(i64 N, const i64* __restrict__ ptr, const int32_t* __restrict__ row,
                                 const double* __restrict__ val, const int32_t* __restrict__ s2g, i64 n,
                                 double* __restrict__ dense) {
  const i64 c = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (c >= N) return;
  const i64 gc = s2g[c];
  for (i64 e = ptr[c]; e < ptr[c + 1]; ++e) dense[static_cast<i64>(s2g[row[e]]) * n + gc] = val[e];
}

// C(i, j) = A(i, cols[j]) (n x m), W(i, j) = A(cols[i], cols[j]) (m x m).
__global__ void k_gather_cw(i64 n, int m, const double* __restrict__ A, const int32_t* __restrict__ cols,
                            double* __restrict__ C, double* __restrict__ W) {
  const i64 x = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (x < n * m) {
    const i64 i = x / m, j = x % m;
    C[x] = A[i * n + cols[j]];
  }
  if (x < static_cast<i64>(m) * m) {
    const i64 i = x / m, j = x % m;
    W[x] = A[static_cast<i64>(cols[i]) * n + cols[j]];
  }
}

// W^+(i, j) = sum over kept e ascending of (inv_e * V(i, e)) * V(j, e), from 0.0
// (transform_ops.hpp:286-294).
__global__ void k_pinv(int m, const double* __restrict__ V, const double* __restrict__ inv,
                       const uint8_t* __restrict__ keep, double* __restrict__ P) {
  const i64 x = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (x >= static_cast<i64>(m) * m) return;
  const i64 i = x / m, j = x % m;
  double acc = 0.0;
  for (int e = 0; e < m; ++e)
    if (keep[e]) acc = dadd(acc, dmul(dmul(inv[e], V[i * m + e]), V[j * m + e]));
  P[x] = acc;
}

// DenseMatrix::multiply (dense.hpp:55-65): out(i, j) = sum over k ascending of
// A(i, k) * B(k, j), terms with A(i, k) == 0 skipped, from 0.0.  A is
// row-major (lda); B(k, j) = Bp[k * bk + j * bj].  64 x 64 output tile per
// CTA, 4 x 4 per thread, 16-deep k chunks staged in shared memory.  With D
// given, writes (D - out)^2 instead (the Frobenius terms).
constexpr int kGT = 64, kGK = 16;
__global__ void __launch_bounds__(256) k_gemm_seq(int M, int N, int K, const double* __restrict__ A, i64 lda,
                                                  const double* __restrict__ B, i64 bk, i64 bj, double* __restrict__ C,
                                                  i64 ldc, const double* __restrict__ D) {
  __shared__ double sa[kGK][kGT + 1], sb[kGK][kGT + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const i64 i0 = static_cast<i64>(blockIdx.y) * kGT, j0 = static_cast<i64>(blockIdx.x) * kGT;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int k0 = 0; k0 < K; k0 += kGK) {
    for (int x = threadIdx.x; x < kGK * kGT; x += 256) {
      const int kk = x % kGK, ii = x / kGK;  // A tile: rows ii, k kk
      const i64 gi = i0 + ii, gk = k0 + kk;
      sa[kk][ii] = (gi < M && gk < K) ? A[gi * lda + gk] : 0.0;
      const int jj = x % kGT, kb = x / kGT;  // B tile: k kb, cols jj
      const i64 gj = j0 + jj, gk2 = k0 + kb;
      sb[kb][jj] = (gj < N && gk2 < K) ? B[gk2 * bk + gj * bj] : 0.0;
    }
    __syncthreads();
    const int kc = min(kGK, K - k0);
    for (int kk = 0; kk < kc; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = sa[kk][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = sb[kk][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        if (av[a] == 0.0) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = dadd(acc[a][b], dmul(av[a], bv[b]));
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const i64 gi = i0 + ty + 16 * a, gj = j0 + tx + 16 * b;
      if (gi >= M || gj >= N) continue;
      if (D) {
        const double d = dsub(D[gi * ldc + gj], acc[a][b]);
        C[gi * ldc + gj] = dmul(d, d);
      } else {
        C[gi * ldc + gj] = acc[a][b];
      }
    }
}

// s = sum of the n*n terms in row-major order, one running sum (the
// reference's double loop, transform_ops.hpp:297-303): lanes load 32
// consecutive terms, lane 0 adds them in order.
__global__ void k_seq_sum(i64 m, const double* __restrict__ t, double* __restrict__ out) {
  const int lane = threadIdx.x;
  double s = 0.0;
  for (i64 b = 0; b < m; b += 32) {
    const double v = b + lane < m ? t[b + lane] : 0.0;
    const int cnt = static_cast<int>((m - b < 32 ? m - b : 32));
    for (int q = 0; q < cnt; ++q) {
      const double w = __shfl_sync(0xffffffffu, v, q);
      s = dadd(s, w);
    }
  }
  if (lane == 0) *out = s;
}

}  // namespace

extern "C" {

int pmmf_b200_precond_create(const pmmf_b200_coo* a, int32_t kind, double omega, void** out, char* err,
                             size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!out) fail(PMMF_INVALID_ARGUMENT, "preconditioner: null output");
    *out = make_precond(a, kind, omega).release();
  });
}

int pmmf_b200_precond_from_operator(void* op, void** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!op || !out) fail(PMMF_INVALID_ARGUMENT, "pmmf_preconditioner: null argument");
    *out = precond_from_operator(op).release();
  });
}

int pmmf_b200_precond_apply(void* pcv, int32_t side, int64_t nrhs, const double* in, double* out, int32_t on_device,
                            char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!pcv) fail(PMMF_INVALID_ARGUMENT, "preconditioner: null handle");
    if (side != 0 && side != 1) fail(PMMF_INVALID_ARGUMENT, "preconditioner: side must be 0 (K^-1) or 1 (K^-T)");
    if (nrhs < 1) return;
    auto* pc = static_cast<SplitPrecond*>(pcv);
    PMMF_CUDA(cudaSetDevice(pc->device));
    if (on_device) PMMF_CUDA(cudaDeviceSynchronize());  // ordered after the caller's producers
    Stream st;
    cudaStream_t s = st.s;
    const i64 n = pc->n, m = n * nrhs;
    if (m == 0) return;
    DBuf<double> a(m, s), b(m, s), c(m, s);
    if (on_device)
      PMMF_CUDA(cudaMemcpyAsync(a.get(), in, sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
    else
      a.upload(in, m);
    to_index_major(a.get(), b.get(), n, static_cast<int>(nrhs), s);
    pc->apply(side, static_cast<int>(nrhs), b.get(), c.get(), s);
    to_rhs_major(c.get(), a.get(), n, static_cast<int>(nrhs), s);
    if (on_device)
      PMMF_CUDA(cudaMemcpyAsync(out, a.get(), sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
    else
      a.download(out, m);
    PMMF_CUDA(cudaStreamSynchronize(s));
  });
}

int pmmf_b200_precond_info(void* pcv, int32_t* kind, int32_t* compensated, double* alpha) {
  if (!pcv) return PMMF_INVALID_ARGUMENT;
  auto* pc = static_cast<SplitPrecond*>(pcv);
  if (kind) *kind = pc->kind;
  if (compensated) *compensated = pc->compensated;
  if (alpha) *alpha = pc->alpha;
  return PMMF_OK;
}

void pmmf_b200_precond_free(void* pcv) { delete static_cast<SplitPrecond*>(pcv); }

int pmmf_b200_solve_precond(const pmmf_b200_coo* a, void* pc, const pmmf_b200_solve_config* cfg, int32_t* iterations,
                            int32_t* converged, int32_t* breakdown, double* residuals, double* wall_ms, char* err,
                            size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!a || !cfg) fail(PMMF_INVALID_ARGUMENT, "solve: null argument");
    run_cg(a, static_cast<SplitPrecond*>(pc), cfg, iterations, converged, breakdown, residuals, wall_ms);
  });
}

int pmmf_b200_nystrom_uniform(const pmmf_b200_coo* a, int64_t m, uint64_t seed, int64_t cap, double* frobenius_error,
                              int64_t* columns, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!a || !frobenius_error || !columns) fail(PMMF_INVALID_ARGUMENT, "nystrom_uniform: null argument");
    const i64 n = a->n;
    if (m < 1 || m > n) fail(PMMF_INVALID_ARGUMENT, "nystrom_uniform: m out of range");
    if (n > cap) fail(PMMF_NUMERIC, "dense_from_blocked: dimension exceeds cap");
    PMMF_CUDA(cudaSetDevice(a->device));
    Stream st;
    cudaStream_t s = st.s;
    // the matrix (from_triplets with the input partition) densely
    Numbering nb;
    {
      std::vector<std::vector<i64>> init;
      if (a->n_clusters == 0) {
        init.emplace_back(static_cast<size_t>(n));
        std::iota(init[0].begin(), init[0].end(), i64{0});
      } else {
        for (i64 u = 0; u < a->n_clusters; ++u)
          init.emplace_back(a->cluster_members + a->cluster_offsets[u],
                            a->cluster_members + a->cluster_offsets[u + 1]);
      }
      nb.build(init, n, s);
    }
    Csc A;
    {
      const int64_t* rows = a->rows;
      const int64_t* cols = a->cols;
      const double* vals = a->vals;
      DBuf<int64_t> dr, dc;
      DBuf<double> dv;
      if (!a->on_device && a->nnz > 0) {
        dr.alloc(a->nnz, s);
        dc.alloc(a->nnz, s);
        dv.alloc(a->nnz, s);
        dr.upload(a->rows, a->nnz);
        dc.upload(a->cols, a->nnz);
        dv.upload(a->vals, a->nnz);
        rows = dr.get();
        cols = dc.get();
        vals = dv.get();
      }
      csc_from_coo(A, nb, n, a->nnz, rows, cols, vals, s, true);
    }
    DBuf<double> dense(n * n, s);
    dense.zero();
    PMMF_LAUNCH(k_dense_from_csc, blocks_for(A.N, kThreads), kThreads, 0, s, A.N, A.ptr.get(), A.row.get(),
                A.val.get(), nb.d_s2g.get(), n, dense.get());
    // m distinct columns (transform_ops.hpp:265-274): the draws stay on the
    // host, like the clustering's anchor draws
    std::vector<i64> ids(static_cast<size_t>(n));
    std::iota(ids.begin(), ids.end(), i64{0});
    Xoshiro rng(seed);
    for (i64 t = 0; t < m; ++t) {
      const i64 pick = t + static_cast<i64>(rng.uniform_below(static_cast<uint64_t>(n - t)));
      std::swap(ids[static_cast<size_t>(t)], ids[static_cast<size_t>(pick)]);
    }
    std::vector<i64> sel(ids.begin(), ids.begin() + m);
    std::sort(sel.begin(), sel.end());
    std::copy(sel.begin(), sel.end(), columns);
    std::vector<int32_t> sel32(sel.begin(), sel.end());
    DBuf<int32_t> dsel(m, s);
    dsel.upload(sel32);
    DBuf<double> C(n * m, s), W(m * m, s), vals(m, s), V(m * m, s), P(m * m, s), CP(n * m, s);
    PMMF_LAUNCH(k_gather_cw, blocks_for(std::max(n * m, m * m), kThreads), kThreads, 0, s, n, static_cast<int>(m),
                dense.get(), dsel.get(), C.get(), W.get());
    eigensystem_dev(static_cast<int>(m), W.get(), vals.get(), V.get(), s);
    const std::vector<double> lam = vals.to_host(m);
    double max_mag = 0.0;
    for (double l : lam) max_mag = std::max(max_mag, std::abs(l));
    const double threshold = 1e-10 * max_mag;
    std::vector<double> inv(static_cast<size_t>(m), 0.0);
    std::vector<uint8_t> keep(static_cast<size_t>(m), 0);
    for (i64 e = 0; e < m; ++e)
      if (!(std::abs(lam[e]) <= threshold)) {
        keep[e] = 1;
        inv[e] = 1.0 / lam[e];
      }
    DBuf<double> dinv(m, s);
    DBuf<uint8_t> dkeep(m, s);
    dinv.upload(inv);
    dkeep.upload(keep);
    PMMF_LAUNCH(k_pinv, blocks_for(m * m, kThreads), kThreads, 0, s, static_cast<int>(m), V.get(), dinv.get(),
                dkeep.get(), P.get());
    // C W^+ (n x m), then (C W^+) C^T against the dense matrix (n x n terms)
    {
      dim3 g(static_cast<unsigned>((m + kGT - 1) / kGT), static_cast<unsigned>((n + kGT - 1) / kGT));
      k_gemm_seq<<<g, 256, 0, s>>>(static_cast<int>(n), static_cast<int>(m), static_cast<int>(m), C.get(), m, P.get(),
                                   m, 1, CP.get(), m, nullptr);
      launch_counter().fetch_add(1, std::memory_order_relaxed);
      PMMF_CUDA(cudaGetLastError());
    }
    DBuf<double> terms(n * n, s), total(1, s);
    {
      dim3 g(static_cast<unsigned>((n + kGT - 1) / kGT), static_cast<unsigned>((n + kGT - 1) / kGT));
      k_gemm_seq<<<g, 256, 0, s>>>(static_cast<int>(n), static_cast<int>(n), static_cast<int>(m), CP.get(), m, C.get(),
                                   1, m, terms.get(), n, dense.get());
      launch_counter().fetch_add(1, std::memory_order_relaxed);
      PMMF_CUDA(cudaGetLastError());
    }
    PMMF_LAUNCH(k_seq_sum, 1, 32, 0, s, n * n, terms.get(), total.get());
    *frobenius_error = std::sqrt(total.to_host(1)[0]);
  });
}

}  // extern "C"
}  // namespace pmmf_b200
