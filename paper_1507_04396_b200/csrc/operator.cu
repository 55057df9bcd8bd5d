// operator.cu — MmfOperator (transform_ops.hpp:30-137) and the
// preconditioned CG harness (solver.hpp:112-167, :343-349, :368-416) on the
// device.
//
// apply(mode): v <- Q v (stages first to last), v <- H^(mode) v, v <- Q^T v
// (stages last to first).  Inside a stage, rotations of different clusters
// touch disjoint indices; inside a cluster they are replayed level by level
// (a level = mutually independent rotations), so one CTA per (cluster, rhs
// chunk) stages the cluster's slice of the vectors in shared memory, applies
// all of its levels with __syncthreads between levels and writes the slice
// back: one HBM read + write of the vectors per stage and direction, rotation
// arithmetic bit-identical to rotate_forward / rotate_transposed.
// Vectors are kept index-major (v[i * nrhs + r]) so a rotation touches
// contiguous rhs lanes.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>

#include "engine.cuh"
#include "layout.cuh"
#include "precond.cuh"
#include "result.cuh"
#include "rng.cuh"
#include "rotation.cuh"
#include "shard.cuh"

namespace pmmf_b200 {

int guarded_call(char* err, size_t errlen, void (*fn)(void*), void* ctx);

namespace {

template <typename F>
int guarded(char* err, size_t errlen, F&& f) {
  return guarded_call(err, errlen, [](void* c) { (*static_cast<F*>(c))(); }, &f);
}

constexpr int kThreads = 256;
constexpr size_t kSmemBudget = 200 * 1024;
constexpr size_t kSmemTwoPerSm = 112 * 1024;

// ------------------------------------------------- core eigensystem (device)
// jacobi_eigensystem (dense.hpp:191-199, called by MmfOperator's constructor,
// transform_ops.hpp:34-41) on the g x g core: one CTA runs the cyclic
// Jacobi of rotation.cuh with the per-pair row / column updates strided over
// its threads (CtaLoop); the Frobenius and off-diagonal sums run on thread 0
// in the reference's order, so values and vectors are bit-identical to the
// reference's sequential sweeps.  Matrices live in shared memory up to
// g = 48, else in global scratch.
struct CtaLoop {
  double* slot;  // one shared double for broadcasts
  template <class F>
  __device__ void each(int n, F&& f) const {
    for (int t = threadIdx.x; t < n; t += blockDim.x) f(t);
  }
  __device__ void sync() const { __syncthreads(); }
  __device__ bool leader() const { return threadIdx.x == 0; }
  __device__ double bcast(double v) const {
    if (threadIdx.x == 0) *slot = v;
    __syncthreads();
    const double r = *slot;
    __syncthreads();
    return r;
  }
};

constexpr int kEigSmemMax = 48;  // two 48 x 48 fp64 tiles = 36 KB of static shared memory

__global__ void k_core_eig(int g, const double* __restrict__ core, double* __restrict__ work_a,
                           double* __restrict__ work_q, double* __restrict__ values, double* __restrict__ vectors) {
  __shared__ double slot;
  __shared__ double sa[kEigSmemMax * kEigSmemMax], sq[kEigSmemMax * kEigSmemMax];
  const bool small = g <= kEigSmemMax;
  double* a = small ? sa : work_a;
  double* q = small ? sq : work_q;
  for (int x = threadIdx.x; x < g * g; x += blockDim.x) a[x] = core[x];
  __syncthreads();
  jacobi_diagonalize_g(RowMajor{a, g}, RowMajor{q, g}, g, CtaLoop{&slot});
  __syncthreads();
  for (int i = threadIdx.x; i < g; i += blockDim.x) values[i] = a[static_cast<long long>(i) * g + i];
  // eigenvectors as columns: vectors(a, e) = q(e, a)
  for (long long x = threadIdx.x; x < static_cast<long long>(g) * g; x += blockDim.x) {
    const long long i = x / g, j = x % g;
    vectors[x] = q[j * g + i];
  }
}

double scalar_factor(int mode, double d, double thr) {  // transform_ops.hpp:76-86
  if (mode == PMMF_APPLY_FORWARD) return d;
  if (mode == PMMF_APPLY_INVERSE) return std::abs(d) < thr ? 0.0 : 1.0 / d;
  return d < thr ? 0.0 : 1.0 / std::sqrt(d);
}

// ------------------------------------------------------------- kernels
struct StageDev {
  int64_t nclusters = 0;
  int64_t max_c = 0;
  size_t max_rec_bytes = 0;  // largest cluster's staged records (k_stage_apply_s)
  DBuf<int32_t> members;   // stage partition, global ids
  DBuf<int64_t> coff;      // cluster offsets
  DBuf<int64_t> rot_ptr;   // per cluster [rot_ptr[u], rot_ptr[u+1]) in level order
  DBuf<int64_t> lvl_ptr;   // per cluster level boundaries: lvl_ptr[lvl_base[u] + L]
  DBuf<int64_t> lvl_base;  // per cluster
  DBuf<int32_t> nlev;      // per cluster
  DBuf<int32_t> loc;       // R x k local positions
  DBuf<double> q;          // R x k x k
  std::vector<int64_t> h_coff, h_rot;  // host: cluster offsets, rotations per apply group (sharding)
};

// Sharded apply (SURVEY.md §8(e) "MMF apply: shard by cluster per stage"):
// pack / unpack the vector rows of a contiguous run of a stage's members.
__global__ void k_pack_rows(int64_t j0, int64_t j1, int nrhs, const int32_t* __restrict__ members,
                            const double* __restrict__ V, double* __restrict__ buf) {
  const int64_t x = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t m = (j1 - j0) * nrhs;
  if (x >= m) return;
  const int64_t j = j0 + x / nrhs;
  buf[j * nrhs + x % nrhs] = V[static_cast<int64_t>(members[j]) * nrhs + x % nrhs];
}
__global__ void k_unpack_rows(int64_t nj, int nrhs, const int32_t* __restrict__ members,
                              const double* __restrict__ buf, double* __restrict__ V) {
  const int64_t x = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (x >= nj * nrhs) return;
  const int64_t j = x / nrhs;
  V[static_cast<int64_t>(members[j]) * nrhs + x % nrhs] = buf[x];
}

template <bool kTransposed>
__global__ void k_stage_apply(int k, int nrhs, int rc, const int64_t* __restrict__ coff,
                              const int32_t* __restrict__ members, const int64_t* __restrict__ rot_ptr,
                              const int64_t* __restrict__ lvl_ptr, const int64_t* __restrict__ lvl_base,
                              const int32_t* __restrict__ nlev, const int32_t* __restrict__ loc,
                              const double* __restrict__ qs, double* __restrict__ V, bool smem_ok) {
  extern __shared__ double sm[];
  const int u = blockIdx.x;
  const int r0 = blockIdx.y * rc;
  const int nr = min(rc, nrhs - r0);
  if (rot_ptr[u + 1] == rot_ptr[u] || nr <= 0) return;
  const int64_t off = coff[u];
  const int c = static_cast<int>(coff[u + 1] - off);
  const int L = nlev[u];
  const int64_t* lp = lvl_ptr + lvl_base[u];
  if (smem_ok) {
    for (int64_t i = threadIdx.x; i < static_cast<int64_t>(c) * nr; i += blockDim.x) {
      const int64_t li = i / nr, r = i % nr;
      sm[li * rc + r] = V[static_cast<int64_t>(members[off + li]) * nrhs + r0 + r];
    }
    __syncthreads();
  }
  for (int lv = 0; lv < L; ++lv) {
    const int l = kTransposed ? (L - 1 - lv) : lv;
    const int64_t b = lp[l], e = lp[l + 1];
    for (int64_t i = threadIdx.x; i < (e - b) * nr; i += blockDim.x) {
      const int64_t t = b + i / nr;
      const int r = static_cast<int>(i % nr);
      double vals[kMaxK];
      int64_t addr[kMaxK];
      for (int x = 0; x < k; ++x) {
        const int li = loc[t * k + x];
        addr[x] = smem_ok ? static_cast<int64_t>(li) * rc + r
                          : static_cast<int64_t>(members[off + li]) * nrhs + r0 + r;
        vals[x] = smem_ok ? sm[addr[x]] : V[addr[x]];
      }
      const double* q = qs + t * k * k;
      for (int a = 0; a < k; ++a) {
        double acc = 0.0;
        for (int x = 0; x < k; ++x) acc = dadd(acc, dmul(kTransposed ? q[x * k + a] : q[a * k + x], vals[x]));
        if (smem_ok)
          sm[addr[a]] = acc;
        else
          V[addr[a]] = acc;
      }
    }
    __syncthreads();
  }
  if (smem_ok) {
    for (int64_t i = threadIdx.x; i < static_cast<int64_t>(c) * nr; i += blockDim.x) {
      const int64_t li = i / nr, r = i % nr;
      V[static_cast<int64_t>(members[off + li]) * nrhs + r0 + r] = sm[li * rc + r];
    }
  }
}

// Slice staging: 8 independent loads in flight per thread (the member
// index and the vector element are two dependent global loads).
constexpr int kGatherUnroll = 8;
__device__ __forceinline__ void gather_slice(double* sm, const double* __restrict__ V,
                                             const int32_t* __restrict__ members, int64_t off, int c, int nr, int rc,
                                             int nrhs, int r0) {
  const int n = c * nr;
  for (int base = threadIdx.x; base < n; base += kGatherUnroll * blockDim.x) {
    int64_t src[kGatherUnroll];
#pragma unroll
    for (int j = 0; j < kGatherUnroll; ++j) {
      const int i = base + j * blockDim.x;
      if (i < n) {
        const int li = i / nr;
        src[j] = static_cast<int64_t>(members[off + li]) * nrhs + r0 + (i - li * nr);
      }
    }
    double x[kGatherUnroll];
#pragma unroll
    for (int j = 0; j < kGatherUnroll; ++j)
      if (base + j * blockDim.x < n) x[j] = V[src[j]];
#pragma unroll
    for (int j = 0; j < kGatherUnroll; ++j) {
      const int i = base + j * blockDim.x;
      if (i < n) {
        const int li = i / nr;
        sm[li * rc + (i - li * nr)] = x[j];
      }
    }
  }
}
template <typename T>
__device__ __forceinline__ void copy_unrolled(T* dst, const T* __restrict__ src, int n) {
  for (int base = threadIdx.x; base < n; base += kGatherUnroll * blockDim.x) {
    T x[kGatherUnroll];
#pragma unroll
    for (int j = 0; j < kGatherUnroll; ++j)
      if (base + j * blockDim.x < n) x[j] = src[base + j * blockDim.x];
#pragma unroll
    for (int j = 0; j < kGatherUnroll; ++j)
      if (base + j * blockDim.x < n) dst[base + j * blockDim.x] = x[j];
  }
}
__device__ __forceinline__ void scatter_slice(const double* sm, double* __restrict__ V,
                                              const int32_t* __restrict__ members, int64_t off, int c, int nr, int rc,
                                              int nrhs, int r0) {
  const int n = c * nr;
  for (int base = threadIdx.x; base < n; base += kGatherUnroll * blockDim.x) {
    int64_t dst[kGatherUnroll];
#pragma unroll
    for (int j = 0; j < kGatherUnroll; ++j) {
      const int i = base + j * blockDim.x;
      if (i < n) {
        const int li = i / nr;
        dst[j] = static_cast<int64_t>(members[off + li]) * nrhs + r0 + (i - li * nr);
      }
    }
#pragma unroll
    for (int j = 0; j < kGatherUnroll; ++j) {
      const int i = base + j * blockDim.x;
      if (i < n) {
        const int li = i / nr;
        V[dst[j]] = sm[li * rc + (i - li * nr)];
      }
    }
  }
}

// Fast path for k = 2, 3 (configs 1-5): same arithmetic as k_stage_apply,
// but the rotation record (local positions + q) of a thread's first item in
// the NEXT level is loaded into registers before the current level's work,
// so the dependent global loads overlap the level instead of following its
// barrier.  The slice always lives in shared memory (run_stage sizes rc).
template <int K, bool kTransposed>
__global__ void __launch_bounds__(256) k_stage_apply_k(int nrhs, int rc, const int64_t* __restrict__ coff,
                                                       const int32_t* __restrict__ members,
                                                       const int64_t* __restrict__ rot_ptr,
                                                       const int64_t* __restrict__ lvl_ptr,
                                                       const int64_t* __restrict__ lvl_base,
                                                       const int32_t* __restrict__ nlev,
                                                       const int32_t* __restrict__ loc,
                                                       const double* __restrict__ qs, double* __restrict__ V) {
  extern __shared__ double sm[];
  const int u = blockIdx.x;
  const int r0 = blockIdx.y * rc;
  const int nr = min(rc, nrhs - r0);
  if (rot_ptr[u + 1] == rot_ptr[u] || nr <= 0) return;
  const int64_t off = coff[u];
  const int c = static_cast<int>(coff[u + 1] - off);
  const int L = nlev[u];
  const int64_t* lp = lvl_ptr + lvl_base[u];
  gather_slice(sm, V, members, off, c, nr, rc, nrhs, r0);
  struct Rec {
    int a[K];
    double q[K * K];
  };
  auto fetch = [&](int64_t t, Rec& x) {
#pragma unroll
    for (int j = 0; j < K; ++j) x.a[j] = loc[t * K + j];
#pragma unroll
    for (int j = 0; j < K * K; ++j) x.q[j] = qs[t * K * K + j];
  };
  auto rotate = [&](const Rec& x, int r) {
    double v[K];
#pragma unroll
    for (int j = 0; j < K; ++j) v[j] = sm[x.a[j] * rc + r];
#pragma unroll
    for (int a = 0; a < K; ++a) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < K; ++j) acc = dadd(acc, dmul(kTransposed ? x.q[j * K + a] : x.q[a * K + j], v[j]));
      sm[x.a[a] * rc + r] = acc;
    }
  };
  auto level_range = [&](int lv, int64_t& b, int64_t& e) {
    const int l = kTransposed ? (L - 1 - lv) : lv;
    b = lp[l];
    e = lp[l + 1];
  };
  Rec cur, nxt;
  int64_t b, e;
  level_range(0, b, e);
  bool have = threadIdx.x < (e - b) * nr;
  if (have) fetch(b + threadIdx.x / nr, cur);
  __syncthreads();
  for (int lv = 0; lv < L; ++lv) {
    int64_t nb = 0, ne = 0;
    bool nhave = false;
    if (lv + 1 < L) {
      level_range(lv + 1, nb, ne);
      nhave = threadIdx.x < (ne - nb) * nr;
      if (nhave) fetch(nb + threadIdx.x / nr, nxt);
    }
    if (have) rotate(cur, threadIdx.x % nr);
    for (int64_t i = threadIdx.x + blockDim.x; i < (e - b) * nr; i += blockDim.x) {  // wide levels
      Rec x;
      fetch(b + i / nr, x);
      rotate(x, static_cast<int>(i % nr));
    }
    __syncthreads();
    cur = nxt;
    have = nhave;
    b = nb;
    e = ne;
  }
  scatter_slice(sm, V, members, off, c, nr, rc, nrhs, r0);
}

// Fully staged variant: the cluster's rotation records (local positions,
// q) and level boundaries are copied into shared memory next to the slice,
// so a level is shared-memory work plus one barrier -- no global load on the
// level chain.  Used when slice + records fit (run_stage).
// Raises a kernel's dynamic shared memory limit only when it grows: a
// captured CG iteration (CUDA graph) then makes no attribute calls.
inline void set_max_smem(const void* kern, size_t bytes) {
  static std::mutex mu;
  static std::map<const void*, size_t> done;
  std::lock_guard<std::mutex> g(mu);
  size_t& cur = done[kern];
  if (bytes <= cur) return;
  PMMF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
  cur = bytes;
}

// 1024 threads: a level's (rotation, rhs) pairs are spread 4x finer than
// over 256, and the level chain's barriers are the critical path (one CTA
// per SM: the slice and records fill shared memory).
constexpr int kApplyThreads = 1024;
template <int K, bool kTransposed>
__global__ void __launch_bounds__(kApplyThreads, 1) k_stage_apply_s(int nrhs, int rc, const int64_t* __restrict__ coff,
                                                       const int32_t* __restrict__ members,
                                                       const int64_t* __restrict__ rot_ptr,
                                                       const int64_t* __restrict__ lvl_ptr,
                                                       const int64_t* __restrict__ lvl_base,
                                                       const int32_t* __restrict__ nlev,
                                                       const int32_t* __restrict__ loc,
                                                       const double* __restrict__ qs, double* __restrict__ V) {
  extern __shared__ double sm[];
  const int u = blockIdx.x;
  const int r0 = blockIdx.y * rc;
  const int nr = min(rc, nrhs - r0);
  const int64_t t0 = rot_ptr[u];
  const int R = static_cast<int>(rot_ptr[u + 1] - t0);
  if (R == 0 || nr <= 0) return;
  const int64_t off = coff[u];
  const int c = static_cast<int>(coff[u + 1] - off);
  const int L = nlev[u];
  const int64_t* lp = lvl_ptr + lvl_base[u];
  double* sq = sm + static_cast<int64_t>(c) * rc;                        // R x K x K
  int* sl = reinterpret_cast<int*>(sq + static_cast<int64_t>(R) * K * K);  // R x K
  int* slp = sl + R * K;                                                   // L + 1
  gather_slice(sm, V, members, off, c, nr, rc, nrhs, r0);
  copy_unrolled(sq, qs + t0 * K * K, R * K * K);
  copy_unrolled(sl, loc + t0 * K, R * K);
  for (int i = threadIdx.x; i <= L; i += blockDim.x) slp[i] = static_cast<int>(lp[i] - t0);
  __syncthreads();
  for (int lv = 0; lv < L; ++lv) {
    const int l = kTransposed ? (L - 1 - lv) : lv;
    const int b = slp[l], n = (slp[l + 1] - b) * nr;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int t = b + i / nr, r = i % nr;
      int a[K];
      double v[K];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        a[j] = sl[t * K + j] * rc + r;
        v[j] = sm[a[j]];
      }
      const double* q = sq + t * K * K;
#pragma unroll
      for (int x = 0; x < K; ++x) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < K; ++j) acc = dadd(acc, dmul(kTransposed ? q[j * K + x] : q[x * K + j], v[j]));
        sm[a[x]] = acc;
      }
    }
    __syncthreads();
  }
  scatter_slice(sm, V, members, off, c, nr, rc, nrhs, r0);
}

// Core: y = E f(lambda) E^T x on the core indices (transform_ops.hpp:88-106),
// one CTA per rhs.
__global__ void k_core_apply(int64_t g, int nrhs, const int32_t* __restrict__ cidx, const double* __restrict__ E,
                             const double* __restrict__ f, double* __restrict__ V) {
  extern __shared__ double sm[];
  double* x = sm;
  double* dot = sm + g;
  const int r = blockIdx.x;
  for (int64_t a = threadIdx.x; a < g; a += blockDim.x) x[a] = V[static_cast<int64_t>(cidx[a]) * nrhs + r];
  __syncthreads();
  for (int64_t e = threadIdx.x; e < g; e += blockDim.x) {
    double d = 0.0;
    for (int64_t a = 0; a < g; ++a) d = dadd(d, dmul(E[a * g + e], x[a]));
    dot[e] = dmul(d, f[e]);
  }
  __syncthreads();
  for (int64_t a = threadIdx.x; a < g; a += blockDim.x) {
    double y = 0.0;
    for (int64_t e = 0; e < g; ++e) y = dadd(y, dmul(E[a * g + e], dot[e]));
    V[static_cast<int64_t>(cidx[a]) * nrhs + r] = y;
  }
}

// Retired diagonal powers: V[idx[d], r] *= f[d].  A warp row per retired
// index, lanes over the rhs (contiguous in the index-major layout): no
// 64-bit division per element (it made this scaling ALU-bound, 3.7x its
// HBM time).
__global__ void k_diag_scale(int64_t nd, int nrhs, const int32_t* __restrict__ idx, const double* __restrict__ f,
                             double* __restrict__ V) {
  const int64_t d = blockIdx.x * static_cast<int64_t>(blockDim.y) + threadIdx.y;
  if (d >= nd) return;
  const double fd = f[d];
  double* row = V + static_cast<int64_t>(idx[d]) * nrhs;
  for (int r = threadIdx.x; r < nrhs; r += 32) row[r] = dmul(row[r], fd);
}


}  // namespace

// ============================================================== Operator
__global__ void k_dense_scatter_coo(int64_t nnz, int64_t n, const int64_t* __restrict__ r,
                                    const int64_t* __restrict__ c, const double* __restrict__ v,
                                    double* __restrict__ A, int* __restrict__ bad) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= nnz) return;
  if (r[t] < 0 || r[t] >= n || c[t] < 0 || c[t] >= n) {
    atomicExch(bad, 1);
    return;
  }
  atomicAdd(A + r[t] * n + c[t], v[t]);
}

// index-major n x cnt block of unit vectors e_{j0 + r}
__global__ void k_unit_block(int64_t n, int cnt, int64_t j0, double* __restrict__ V) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= n * cnt) return;
  const int64_t i = t / cnt, r = t % cnt;
  V[t] = i == j0 + r ? 1.0 : 0.0;
}

// per-block partial sums of (A[i][j0+r] - V[i][r])^2 over the batch
__global__ void k_diff_sq(int64_t n, int cnt, int64_t j0, const double* __restrict__ A, const double* __restrict__ V,
                          double* __restrict__ part) {
  extern __shared__ double red[];
  double acc = 0.0;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n * cnt;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = t / cnt, r = t % cnt;
    const double d = A[i * n + j0 + r] - V[t];
    acc += d * d;
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (static_cast<int>(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

struct Operator {
  int device = 0;
  int64_t n = 0;
  int k = 2;
  double thr = 1e-12;
  int64_t neg = 0;
  std::vector<StageDev> stages;
  int64_t g = 0;
  DBuf<int32_t> core_idx;
  DBuf<double> E;
  DBuf<double> core_f[3];
  int64_t nd = 0;
  DBuf<int32_t> diag_idx;
  DBuf<double> diag_f[3];
  cudaStream_t s = nullptr;

  ~Operator() {
    stages.clear();
    core_idx.release();
    E.release();
    for (auto& x : core_f) x.release();
    diag_idx.release();
    for (auto& x : diag_f) x.release();
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }

  void build(const Result& f) {
    PMMF_CUDA(cudaGetDevice(&device));
    PMMF_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    n = f.n;
    k = f.k;
    for (const auto& st : f.stages) {
      StageDev sd;
      const int64_t m = static_cast<int64_t>(st.off.size()) - 1;
      sd.nclusters = m;
      std::vector<int64_t> pos_of(static_cast<size_t>(n), -1), cl_of(static_cast<size_t>(n), -1);
      for (int64_t u = 0; u < m; ++u) {
        sd.max_c = std::max<int64_t>(sd.max_c, st.off[u + 1] - st.off[u]);
        for (int64_t i = st.off[u]; i < st.off[u + 1]; ++i) {
          pos_of[st.members[i]] = i - st.off[u];
          cl_of[st.members[i]] = u;
        }
      }
      const int64_t R = static_cast<int64_t>(st.rot_idx.size()) / k;
      // per cluster: non-identity rotations with their dependency level
      std::vector<std::vector<std::pair<int32_t, int64_t>>> per(static_cast<size_t>(m));  // (level, t)
      std::vector<int32_t> lastlvl(static_cast<size_t>(n), 0);
      for (int64_t t = 0; t < R; ++t) {
        const double* q = st.rot_q.data() + t * k * k;
        bool ident = true;
        for (int a = 0; a < k; ++a)
          for (int b = 0; b < k; ++b) ident = ident && q[a * k + b] == (a == b ? 1.0 : 0.0);
        if (ident) continue;  // value-neutral
        const int64_t u = cl_of[st.rot_idx[t * k]];
        if (u < 0) fail(PMMF_INVALID_ARGUMENT, "MmfOperator: rotation index not in its stage partition");
        int32_t lv = 0;
        for (int a = 0; a < k; ++a) {
          if (cl_of[st.rot_idx[t * k + a]] != u) fail(PMMF_INVALID_ARGUMENT, "MmfOperator: rotation spans clusters");
          lv = std::max(lv, lastlvl[st.rot_idx[t * k + a]]);
        }
        ++lv;
        for (int a = 0; a < k; ++a) lastlvl[st.rot_idx[t * k + a]] = lv;
        per[u].push_back({lv, t});
      }
      // Apply groups: the clusters with at least one non-identity rotation,
      // each reduced to the indices those rotations touch (identity
      // rotations are 51% of config 5's stage 1 and 98% of its stage 2; an
      // untouched index keeps its value, so it is neither read nor written).
      std::vector<int64_t> rot_ptr(1, 0), lvl_ptr, lvl_base, coff(1, 0);
      std::vector<int32_t> nlev, loc, mem;
      std::vector<double> qv;
      std::vector<int32_t> slot(static_cast<size_t>(sd.max_c), -1);
      sd.max_c = 0;
      for (int64_t u = 0; u < m; ++u) {
        auto& v = per[u];
        if (v.empty()) continue;
        std::stable_sort(v.begin(), v.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
        const size_t mem0 = mem.size();
        lvl_base.push_back(static_cast<int64_t>(lvl_ptr.size()));
        const int32_t L = v.back().first;
        nlev.push_back(L);
        int64_t cur = rot_ptr.back();
        size_t i = 0;
        for (int32_t lv = 1; lv <= L; ++lv) {
          lvl_ptr.push_back(cur);
          while (i < v.size() && v[i].first == lv) {
            const int64_t t = v[i].second;
            for (int a = 0; a < k; ++a) {
              const int64_t gidx = st.rot_idx[t * k + a];
              int32_t& sl = slot[static_cast<size_t>(pos_of[gidx])];
              if (sl < 0) {
                sl = static_cast<int32_t>(mem.size() - mem0);
                mem.push_back(static_cast<int32_t>(gidx));
              }
              loc.push_back(sl);
            }
            qv.insert(qv.end(), st.rot_q.begin() + t * k * k, st.rot_q.begin() + (t + 1) * k * k);
            ++cur;
            ++i;
          }
        }
        for (size_t j = mem0; j < mem.size(); ++j) slot[static_cast<size_t>(pos_of[mem[j]])] = -1;
        lvl_ptr.push_back(cur);
        rot_ptr.push_back(cur);
        coff.push_back(static_cast<int64_t>(mem.size()));
        sd.max_c = std::max<int64_t>(sd.max_c, static_cast<int64_t>(mem.size() - mem0));
        const size_t rb = v.size() * static_cast<size_t>(k * k * 8 + k * 4) + static_cast<size_t>(L + 1) * 4;
        sd.max_rec_bytes = std::max(sd.max_rec_bytes, (rb + 15) / 16 * 16);
      }
      sd.nclusters = static_cast<int64_t>(coff.size()) - 1;
      auto up64 = [&](DBuf<int64_t>& d, const std::vector<int64_t>& h) {
        d.alloc(std::max<int64_t>(1, static_cast<int64_t>(h.size())), s);
        d.upload(h);
      };
      auto up32 = [&](DBuf<int32_t>& d, const std::vector<int32_t>& h) {
        d.alloc(std::max<int64_t>(1, static_cast<int64_t>(h.size())), s);
        d.upload(h);
      };
      up32(sd.members, mem);
      up64(sd.coff, coff);
      up64(sd.rot_ptr, rot_ptr);
      up64(sd.lvl_ptr, lvl_ptr);
      up64(sd.lvl_base, lvl_base);
      up32(sd.nlev, nlev);
      up32(sd.loc, loc);
      sd.h_coff = coff;
      sd.h_rot.resize(static_cast<size_t>(sd.nclusters));
      for (int64_t u = 0; u < sd.nclusters; ++u) sd.h_rot[u] = rot_ptr[u + 1] - rot_ptr[u];
      sd.q.alloc(std::max<int64_t>(1, static_cast<int64_t>(qv.size())), s);
      sd.q.upload(qv);
      PMMF_CUDA(cudaStreamSynchronize(s));
      stages.push_back(std::move(sd));
    }
    // core eigensystem (transform_ops.hpp:34-41) on the device
    g = static_cast<int64_t>(f.core_idx.size());
    std::vector<double> vals;
    if (g > 0) {
      DBuf<double> dcore(g * g, s), dval(g, s);
      E.alloc(g * g, s);
      dcore.upload(f.core);
      DBuf<double> wa, wq;
      if (g > kEigSmemMax) {
        wa.alloc(g * g, s);
        wq.alloc(g * g, s);
      }
      const int threads = g <= 32 ? 32 : (g <= kEigSmemMax ? 64 : 256);
      PMMF_LAUNCH(k_core_eig, 1, threads, 0, s, static_cast<int>(g), dcore.get(), wa.get(), wq.get(), dval.get(),
                  E.get());
      vals = dval.to_host(g);
    }
    for (double l : vals)
      if (l < -thr) ++neg;
    for (const auto& d : f.diag)
      if (d.second < -thr) ++neg;
    if (g > 0) {
      std::vector<int32_t> ci(f.core_idx.begin(), f.core_idx.end());
      core_idx.alloc(g, s);
      core_idx.upload(ci);
      for (int mode = 0; mode < 3; ++mode) {
        std::vector<double> fv(static_cast<size_t>(g));
        for (int64_t e = 0; e < g; ++e) fv[e] = scalar_factor(mode, vals[e], thr);
        core_f[mode].alloc(g, s);
        core_f[mode].upload(fv);
      }
    }
    nd = static_cast<int64_t>(f.diag.size());
    if (nd > 0) {
      std::vector<int32_t> di(static_cast<size_t>(nd));
      for (int64_t i = 0; i < nd; ++i) di[i] = static_cast<int32_t>(f.diag[i].first);
      diag_idx.alloc(nd, s);
      diag_idx.upload(di);
      for (int mode = 0; mode < 3; ++mode) {
        std::vector<double> fv(static_cast<size_t>(nd));
        for (int64_t i = 0; i < nd; ++i) fv[i] = scalar_factor(mode, f.diag[i].second, thr);
        diag_f[mode].alloc(nd, s);
        diag_f[mode].upload(fv);
      }
    }
    PMMF_CUDA(cudaStreamSynchronize(s));
  }

  // Apply groups [u0, u1) of a stage (default all): the kernels index their
  // group by blockIdx.x, so the range is passed as offset per-group arrays.
  void run_stage(const StageDev& sd, bool transposed, int nrhs, double* V, cudaStream_t st, int64_t u0 = 0,
                 int64_t u1 = -1) const {
    if (u1 < 0) u1 = sd.nclusters;
    const int64_t ng = u1 - u0;
    if (ng <= 0) return;
    const int64_t* coff = sd.coff.get() + u0;
    const int64_t* rotp = sd.rot_ptr.get() + u0;
    const int64_t* lbase = sd.lvl_base.get() + u0;
    const int32_t* nlev = sd.nlev.get() + u0;
    if ((k == 2 || k == 3) && sd.max_rec_bytes > 0) {
      // Records staged in shared memory: the widest rhs chunk (<= 8) whose
      // slice fits next to the largest cluster's records.
      const size_t row = static_cast<size_t>(sd.max_c) * 8;
      int rc = std::min(nrhs, 8);
      const size_t cap = row + sd.max_rec_bytes <= kSmemTwoPerSm ? kSmemTwoPerSm : kSmemBudget;
      while (rc > 1 && row * rc + sd.max_rec_bytes > cap) --rc;
      const size_t smem = row * rc + sd.max_rec_bytes;
      if (smem <= kSmemBudget) {
        dim3 grid(static_cast<unsigned>(ng), static_cast<unsigned>((nrhs + rc - 1) / rc));
        auto kern = k == 2 ? (transposed ? k_stage_apply_s<2, true> : k_stage_apply_s<2, false>)
                           : (transposed ? k_stage_apply_s<3, true> : k_stage_apply_s<3, false>);
        if (smem > 48 * 1024)
          set_max_smem(reinterpret_cast<const void*>(kern), smem);
        kern<<<grid, kApplyThreads, smem, st>>>(nrhs, rc, coff, sd.members.get(), rotp, sd.lvl_ptr.get(), lbase,
                                                nlev, sd.loc.get(), sd.q.get(), V);
        launch_counter().fetch_add(1, std::memory_order_relaxed);
        PMMF_CUDA(cudaGetLastError());
        return;
      }
    }
    if (k == 2 || k == 3) {
      // rhs per CTA: as many as fit two CTAs per SM (<= 8), else one CTA
      // per SM with the largest slice that fits.
      const size_t row = static_cast<size_t>(sd.max_c) * 8;
      int rc = std::min(nrhs, 8);
      while (rc > 1 && row * rc > kSmemTwoPerSm) --rc;
      if (row * rc <= kSmemBudget) {
        const size_t smem = row * rc;
        dim3 grid(static_cast<unsigned>(ng), static_cast<unsigned>((nrhs + rc - 1) / rc));
        auto kern = k == 2 ? (transposed ? k_stage_apply_k<2, true> : k_stage_apply_k<2, false>)
                           : (transposed ? k_stage_apply_k<3, true> : k_stage_apply_k<3, false>);
        if (smem > 48 * 1024)
          set_max_smem(reinterpret_cast<const void*>(kern), smem);
        kern<<<grid, kThreads, smem, st>>>(nrhs, rc, coff, sd.members.get(), rotp, sd.lvl_ptr.get(), lbase,
                                           nlev, sd.loc.get(), sd.q.get(), V);
        launch_counter().fetch_add(1, std::memory_order_relaxed);
        PMMF_CUDA(cudaGetLastError());
        return;
      }
    }
    int rc = std::min(nrhs, 8);
    while (rc > 1 && static_cast<size_t>(sd.max_c) * rc * 8 > kSmemBudget) rc >>= 1;
    const bool smem_ok = static_cast<size_t>(sd.max_c) * rc * 8 <= kSmemBudget;
    const size_t smem = smem_ok ? static_cast<size_t>(sd.max_c) * rc * 8 : 0;
    dim3 grid(static_cast<unsigned>(ng), static_cast<unsigned>((nrhs + rc - 1) / rc));
    auto kern = transposed ? k_stage_apply<true> : k_stage_apply<false>;
    if (smem > 48 * 1024) set_max_smem(reinterpret_cast<const void*>(kern), smem);
    kern<<<grid, kThreads, smem, st>>>(k, nrhs, rc, coff, sd.members.get(), rotp, sd.lvl_ptr.get(), lbase, nlev,
                                       sd.loc.get(), sd.q.get(), V, smem_ok);
    launch_counter().fetch_add(1, std::memory_order_relaxed);
    PMMF_CUDA(cudaGetLastError());
  }

  // V: index-major n x nrhs on the device.
  void apply_dev(int mode, int nrhs, double* V, cudaStream_t st) const {
    for (const auto& sd : stages) run_stage(sd, false, nrhs, V, st);
    if (g > 0) {
      const size_t smem = static_cast<size_t>(2 * g) * 8;
      if (smem > 48 * 1024) set_max_smem(reinterpret_cast<const void*>(k_core_apply), smem);
      PMMF_LAUNCH(k_core_apply, static_cast<unsigned>(nrhs), kThreads, smem, st, g, nrhs, core_idx.get(), E.get(),
                  core_f[mode].get(), V);
    }
    if (nd > 0)
      PMMF_LAUNCH(k_diag_scale, static_cast<unsigned>((nd + 7) / 8), dim3(32, 8), 0, st, nd, nrhs, diag_idx.get(),
                  diag_f[mode].get(), V);
    for (auto it = stages.rbegin(); it != stages.rend(); ++it) run_stage(*it, true, nrhs, V, st);
  }

  // apply over W ranks (shard.cuh): stage by stage, rank r applies the
  // rotations of its contiguous range of apply groups (shard_ranges, cost
  // from rotations and group sizes) to the rows it then owns, and the
  // updated rows are exchanged before the next stage (grouped broadcasts of
  // each rank's packed segment; virtual ranks share V).  Core and retired
  // diagonals are applied by every rank.  Same kernels, same order per row:
  // bit-identical to apply_dev for any W.
  void apply_dev_sharded(int mode, int nrhs, double* V, cudaStream_t st, const Comm& C) const {
    const int W = C.world();
    auto split = [&](const StageDev& sd) {
      std::vector<i64> sz(sd.h_rot.begin(), sd.h_rot.end()), c(static_cast<size_t>(sd.nclusters));
      for (int64_t u = 0; u < sd.nclusters; ++u) c[u] = sd.h_coff[u + 1] - sd.h_coff[u];
      return shard_ranges(sz, c, W);
    };
    DBuf<double> buf;
    auto stage = [&](const StageDev& sd, bool transposed) {
      const std::vector<i64> lo = split(sd);
      for (const int r : C.local_ranks()) run_stage(sd, transposed, nrhs, V, st, lo[r], lo[r + 1]);
      if (!C.multi_process()) return;
      const int64_t total = sd.h_coff.back();
      if (buf.n < total * nrhs) buf.alloc(std::max<int64_t>(total * nrhs, 1), st);
      const int64_t j0 = sd.h_coff[lo[C.rank]], j1 = sd.h_coff[lo[C.rank + 1]];
      PMMF_LAUNCH(k_pack_rows, blocks_for((j1 - j0) * nrhs, kThreads), kThreads, 0, st, j0, j1, nrhs,
                  sd.members.get(), V, buf.get());
      std::vector<i64> seg(static_cast<size_t>(W) + 1);
      for (int q = 0; q <= W; ++q) seg[q] = sd.h_coff[lo[q]];
      bcast_segments(buf.get(), sizeof(double) * nrhs, seg, C, st);
      PMMF_LAUNCH(k_unpack_rows, blocks_for(total * nrhs, kThreads), kThreads, 0, st, total, nrhs, sd.members.get(),
                  buf.get(), V);
    };
    for (const auto& sd : stages) stage(sd, false);
    if (g > 0) {
      const size_t smem = static_cast<size_t>(2 * g) * 8;
      if (smem > 48 * 1024) set_max_smem(reinterpret_cast<const void*>(k_core_apply), smem);
      PMMF_LAUNCH(k_core_apply, static_cast<unsigned>(nrhs), kThreads, smem, st, g, nrhs, core_idx.get(), E.get(),
                  core_f[mode].get(), V);
    }
    if (nd > 0)
      PMMF_LAUNCH(k_diag_scale, static_cast<unsigned>((nd + 7) / 8), dim3(32, 8), 0, st, nd, nrhs, diag_idx.get(),
                  diag_f[mode].get(), V);
    for (auto it = stages.rbegin(); it != stages.rend(); ++it) stage(*it, true);
  }
};

// ====================================================== CG (solver.hpp)
namespace {

// y[g(row)*nrhs + r] = sum over the row's columns (input-partition order) of
// a * x, skipping x == 0 (multiply_flat, blocked_matrix.hpp:390-407).
// Warp per row, lane per rhs.
__global__ void k_spmv(int64_t N, int nrhs, const int64_t* __restrict__ ptr, const int32_t* __restrict__ col,
                       const double* __restrict__ val, const int32_t* __restrict__ s2g, const double* __restrict__ X,
                       double* __restrict__ Y) {
  const int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= N) return;
  const int64_t gr = s2g[w];
  for (int r = lane; r < nrhs; r += 32) {
    double acc = 0.0;
    for (int64_t e = ptr[w]; e < ptr[w + 1]; ++e) {
      const double x = X[static_cast<int64_t>(s2g[col[e]]) * nrhs + r];
      if (x == 0.0) continue;
      acc = dadd(acc, dmul(val[e], x));
    }
    Y[gr * nrhs + r] = acc;
  }
}

// Deterministic per-rhs dot products: fixed grid of partials, then a fixed
// order final pass (no atomics).  Vectors are index-major (v[i * nrhs + r]):
// a warp reads one row's rhs lanes contiguously, block b owns a contiguous
// row range, warp w its rows b0 + w + 8k, lane r the running sum of rhs r;
// the 8 warps' sums are folded in warp order.
constexpr int kDotBlocks = 1184;  // 8 per SM: enough loads in flight to stream both vectors
__global__ void __launch_bounds__(kThreads) k_dot_partial(int64_t n, int nrhs, const double* __restrict__ a,
                                                          const double* __restrict__ b, double* __restrict__ part) {
  __shared__ double red[kThreads / 32][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = kThreads / 32;
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t i0 = blockIdx.x * per, i1 = min(n, i0 + per);
  for (int r0 = 0; r0 < nrhs; r0 += 32) {
    const int r = r0 + lane;
    double s = 0.0;
    if (r < nrhs) {
      int64_t i = i0 + w;
      for (; i + 3 * nw < i1; i += 4 * nw) {  // four rows' loads in flight, the sum still in row order
        const double a0 = a[i * nrhs + r], b0 = b[i * nrhs + r];
        const double a1 = a[(i + nw) * nrhs + r], b1 = b[(i + nw) * nrhs + r];
        const double a2 = a[(i + 2 * nw) * nrhs + r], b2 = b[(i + 2 * nw) * nrhs + r];
        const double a3 = a[(i + 3 * nw) * nrhs + r], b3 = b[(i + 3 * nw) * nrhs + r];
        s = dadd(s, dmul(a0, b0));
        s = dadd(s, dmul(a1, b1));
        s = dadd(s, dmul(a2, b2));
        s = dadd(s, dmul(a3, b3));
      }
      for (; i < i1; i += nw) s = dadd(s, dmul(a[i * nrhs + r], b[i * nrhs + r]));
    }
    red[w][lane] = s;
    __syncthreads();
    if (w == 0 && r < nrhs) {
      double t = red[0][lane];
      for (int q = 1; q < nw; ++q) t = dadd(t, red[q][lane]);
      part[static_cast<int64_t>(r) * gridDim.x + blockIdx.x] = t;
    }
    __syncthreads();
  }
}
// Warp per rhs: lanes load 32 partials at a time (coalesced), lane 0 adds
// them in partial order (the same fixed order as a sequential loop).
__global__ void k_dot_final(int nrhs, int nparts, const double* __restrict__ part, double* __restrict__ out) {
  const int r = blockIdx.x, lane = threadIdx.x;
  if (r >= nrhs) return;
  double s = 0.0;
  for (int p0 = 0; p0 < nparts; p0 += 32) {
    const double v = p0 + lane < nparts ? part[static_cast<int64_t>(r) * nparts + p0 + lane] : 0.0;
    const int cnt = nparts - p0 < 32 ? nparts - p0 : 32;
    for (int q = 0; q < cnt; ++q) s = dadd(s, __shfl_sync(0xffffffffu, v, q));
  }
  if (lane == 0) out[r] = s;
}

struct CgState {
  double* rr;
  double* pap;
  double* res;
  double* rrn;
  double* alpha;
  double* bnorm;
  int32_t* active;
  int32_t* iters;
  int32_t* conv;
  int32_t* brk;
  double* trace;
  int stride;
  double tol;
};

__global__ void k_cg_alpha(int nrhs, CgState S) {
  const int r = threadIdx.x;
  if (r >= nrhs || !S.active[r]) return;
  if (!(S.pap[r] > 0.0)) {
    S.brk[r] = 1;
    S.active[r] = 0;
    S.alpha[r] = 0.0;
    return;
  }
  S.alpha[r] = S.rr[r] / S.pap[r];
}
// y += alpha p; r -= alpha w (active rhs only; alpha = 0 otherwise is not used)
__global__ void k_cg_update(int64_t n, int nrhs, const int32_t* __restrict__ active, const double* __restrict__ alpha,
                            const double* __restrict__ p, const double* __restrict__ w, double* __restrict__ y,
                            double* __restrict__ rv) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n * nrhs) return;
  const int r = static_cast<int>(i % nrhs);
  if (!active[r]) return;
  y[i] = dadd(y[i], dmul(alpha[r], p[i]));
  rv[i] = dsub(rv[i], dmul(alpha[r], w[i]));
}
__global__ void k_sub(int64_t m, const double* __restrict__ b, const double* __restrict__ t, double* __restrict__ o) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < m) o[i] = dsub(b[i], t[i]);
}
// The iteration number comes from a device counter (k_cg_tick), so one
// captured iteration can be replayed as a CUDA graph.
__global__ void k_cg_tick(int32_t* it) { ++*it; }
__global__ void k_cg_check(int nrhs, const int32_t* __restrict__ itp, CgState S) {
  const int it = *itp;
  const int r = threadIdx.x;
  if (r >= nrhs || !S.active[r]) return;
  const double res = sqrt(S.res[r]);
  S.trace[static_cast<int64_t>(r) * S.stride + it] = res;
  S.iters[r] = it;
  if (res / S.bnorm[r] <= S.tol) {
    S.conv[r] = 1;
    S.active[r] = 0;
  }
}
__global__ void k_cg_beta(int64_t n, int nrhs, const int32_t* __restrict__ active, const double* __restrict__ rrn,
                          double* __restrict__ rr, const double* __restrict__ rv, double* __restrict__ p) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n * nrhs) return;
  const int r = static_cast<int>(i % nrhs);
  if (!active[r]) return;
  const double beta = rrn[r] / rr[r];
  p[i] = dadd(rv[i], dmul(beta, p[i]));
}
__global__ void k_cg_rr(int nrhs, const int32_t* __restrict__ active, const double* __restrict__ rrn, double* __restrict__ rr) {
  const int r = threadIdx.x;
  if (r < nrhs && active[r]) rr[r] = rrn[r];
}

}  // namespace

void eigensystem_dev(int g, const double* a, double* values, double* vectors, cudaStream_t s) {
  if (g <= 0) return;
  DBuf<double> wa, wq;
  if (g > kEigSmemMax) {
    wa.alloc(static_cast<int64_t>(g) * g, s);
    wq.alloc(static_cast<int64_t>(g) * g, s);
  }
  const int threads = g <= 32 ? 32 : (g <= kEigSmemMax ? 64 : 256);
  PMMF_LAUNCH(k_core_eig, 1, threads, 0, s, g, a, wa.get(), wq.get(), values, vectors);
  PMMF_CUDA(cudaStreamSynchronize(s));
}

namespace {
// pmmf_preconditioner (solver.hpp:343-349): both sides are apply(inv_sqrt).
struct OpPrecond : SplitPrecond {
  const Operator* op = nullptr;
  void apply(int, int nr, const double* in, double* out, cudaStream_t s) override {
    PMMF_CUDA(cudaMemcpyAsync(out, in, sizeof(double) * n * nr, cudaMemcpyDeviceToDevice, s));
    op->apply_dev(PMMF_APPLY_INV_SQRT, nr, out, s);
  }
};
}  // namespace

std::unique_ptr<SplitPrecond> precond_from_operator(void* opv) {
  const auto* o = static_cast<const Operator*>(opv);
  PMMF_CUDA(cudaSetDevice(o->device));
  auto p = std::make_unique<OpPrecond>();
  p->kind = PMMF_PRECOND_PMMF;
  p->op = o;
  p->n = o->n;
  p->device = o->device;
  return p;
}

// run_solve_experiment (solver.hpp:368-416) over pcg_symmetric
// (solver.hpp:112-167): all rhs_count right-hand sides advance together.
void run_cg(const pmmf_b200_coo* a, SplitPrecond* pc, const pmmf_b200_solve_config* cfg, int32_t* iterations,
            int32_t* converged, int32_t* breakdown, double* residuals, double* wall_ms) {
    if (!(cfg->tol > 0.0)) fail(PMMF_INVALID_ARGUMENT, "SolveConfig: tol must be positive");
    if (cfg->max_iter < 1) fail(PMMF_INVALID_ARGUMENT, "SolveConfig: max_iter < 1");
    if (cfg->rhs_count < 1) fail(PMMF_INVALID_ARGUMENT, "SolveConfig: rhs_count < 1");
    if (cfg->rhs_count > 1024) fail(PMMF_INVALID_ARGUMENT, "SolveConfig: rhs_count > 1024 unsupported");
    PMMF_CUDA(cudaSetDevice(a->device));
    cudaStream_t s;
    PMMF_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct SG {
      cudaStream_t s;
      ~SG() {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
      }
    } sg{s};
    const auto start = std::chrono::steady_clock::now();
    const int64_t n = a->n;
    const int nr = cfg->rhs_count;
    if (pc && pc->n != n) fail(PMMF_INVALID_ARGUMENT, "pcg_symmetric: operator dimension mismatch");
    if (pc && pc->device != a->device) fail(PMMF_INVALID_ARGUMENT, "pcg_symmetric: preconditioner on another device");
    // Matrix rows in input-partition order for y = A x.
    Numbering nb;
    {
      std::vector<std::vector<int64_t>> init;
      if (a->n_clusters == 0) {
        init.emplace_back(static_cast<size_t>(n));
        std::iota(init[0].begin(), init[0].end(), int64_t{0});
      } else {
        for (int64_t u = 0; u < a->n_clusters; ++u)
          init.emplace_back(a->cluster_members + a->cluster_offsets[u], a->cluster_members + a->cluster_offsets[u + 1]);
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
      csc_from_coo(A, nb, n, a->nnz, rows, cols, vals, s);
    }
    Csc Arow;  // transpose: per row (stage id), columns ascending in stage order
    {
      Paged P;
      const int64_t nz = A.nnz;
      paged_from_csc(P, std::move(A), 1, s);
      (void)nz;
      transpose_paged(Arow, P, s);
    }
    // right-hand sides (solver.hpp:375-381), bnorm on the host in order
    std::vector<double> hb(static_cast<size_t>(n * nr)), bimaj(static_cast<size_t>(n * nr)), bn(static_cast<size_t>(nr));
    for (int r = 0; r < nr; ++r) {
      const uint64_t path[2] = {0xB0u, static_cast<uint64_t>(r)};
      Xoshiro rng(derive(cfg->seed, path));
      double* b = hb.data() + static_cast<int64_t>(r) * n;
      for (int64_t i = 0; i < n; ++i) b[i] = normal_draw(rng);
      double sq = 0.0;
      for (int64_t i = 0; i < n; ++i) sq += b[i] * b[i];
      const double norm = std::sqrt(sq);
      if (norm > 0.0)
        for (int64_t i = 0; i < n; ++i) b[i] /= norm;
      double s2 = 0.0;
      for (int64_t i = 0; i < n; ++i) s2 += b[i] * b[i];
      bn[r] = std::sqrt(s2);
      for (int64_t i = 0; i < n; ++i) bimaj[i * nr + r] = b[i];
    }
    const int stride = cfg->max_iter + 1;
    for (int64_t i = 0; i < static_cast<int64_t>(nr) * stride; ++i) residuals[i] = NAN;
    std::vector<int32_t> act(static_cast<size_t>(nr), 1), zero(static_cast<size_t>(nr), 0);
    for (int r = 0; r < nr; ++r) {
      residuals[static_cast<int64_t>(r) * stride] = bn[r];
      iterations[r] = 0;
      converged[r] = 0;
      breakdown[r] = 0;
      if (bn[r] == 0.0) {
        converged[r] = 1;
        act[r] = 0;
      }
    }
    const int64_t m = n * nr;
    DBuf<double> B(m, s), Y(m, s), Rv(m, s), Pv(m, s), W(m, s), T1(m, s), T2(m, s), X(m, s);
    B.upload(bimaj);
    Y.zero();
    DBuf<double> part(static_cast<int64_t>(kDotBlocks) * nr, s);
    DBuf<double> rr(nr, s), pap(nr, s), res(nr, s), rrn(nr, s), alpha(nr, s), dbn(nr, s);
    DBuf<int32_t> dact(nr, s), diters(nr, s), dconv(nr, s), dbrk(nr, s);
    DBuf<double> trace(static_cast<int64_t>(nr) * stride, s);
    dbn.upload(bn);
    dact.upload(act);
    diters.upload(zero);
    dconv.upload(zero);
    dbrk.upload(zero);
    trace.fill_bytes(0xff);  // NaN pattern
    // side 0: K^-1, side 1: K^-T (identity_preconditioner when pc is null)
    auto pre = [&](int side, const DBuf<double>& in, DBuf<double>& out) {
      if (pc)
        pc->apply(side, nr, in.get(), out.get(), s);
      else
        PMMF_CUDA(cudaMemcpyAsync(out.get(), in.get(), sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
    };
    auto spmv = [&](const DBuf<double>& x, DBuf<double>& y) {
      y.zero();
      PMMF_LAUNCH(k_spmv, blocks_for(Arow.N * 32, kThreads), kThreads, 0, s, Arow.N, nr, Arow.ptr.get(), Arow.row.get(),
                  Arow.val.get(), nb.d_s2g.get(), x.get(), y.get());
    };
    auto dot = [&](const DBuf<double>& x, const DBuf<double>& y, DBuf<double>& out) {
      PMMF_LAUNCH(k_dot_partial, kDotBlocks, kThreads, 0, s, n, nr, x.get(), y.get(), part.get());
      PMMF_LAUNCH(k_dot_final, static_cast<unsigned>(nr), 32, 0, s, nr, kDotBlocks, part.get(), out.get());
    };
    CgState S{rr.get(), pap.get(), res.get(), rrn.get(), alpha.get(), dbn.get(), dact.get(), diters.get(),
              dconv.get(), dbrk.get(), trace.get(), stride, cfg->tol};
    const int th = std::max(32, ((nr + 31) / 32) * 32);
    pre(0, B, Rv);  // r = K^-1 b
    PMMF_CUDA(cudaMemcpyAsync(Pv.get(), Rv.get(), sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
    dot(Rv, Rv, rr);
    DBuf<int32_t> dit(1, s);
    dit.zero();
    auto iteration = [&] {
      PMMF_LAUNCH(k_cg_tick, 1, 1, 0, s, dit.get());
      pre(1, Pv, T1);
      spmv(T1, T2);
      pre(0, T2, W);
      dot(Pv, W, pap);
      PMMF_LAUNCH(k_cg_alpha, 1, th, 0, s, nr, S);
      PMMF_LAUNCH(k_cg_update, blocks_for(m, kThreads), kThreads, 0, s, n, nr, dact.get(), alpha.get(), Pv.get(),
                  W.get(), Y.get(), Rv.get());
      pre(1, Y, X);
      spmv(X, T2);
      PMMF_LAUNCH(k_sub, blocks_for(m, kThreads), kThreads, 0, s, m, B.get(), T2.get(), T1.get());
      dot(T1, T1, res);
      PMMF_LAUNCH(k_cg_check, 1, th, 0, s, nr, dit.get(), S);
      dot(Rv, Rv, rrn);
      PMMF_LAUNCH(k_cg_beta, blocks_for(m, kThreads), kThreads, 0, s, n, nr, dact.get(), rrn.get(), rr.get(), Rv.get(),
                  Pv.get());
      PMMF_LAUNCH(k_cg_rr, 1, th, 0, s, nr, dact.get(), rrn.get(), rr.get());
    };
    auto all_done = [&] {
      std::vector<int32_t> h = dact.to_host(nr);
      for (int r = 0; r < nr; ++r)
        if (h[r]) return false;
      return true;
    };
    // The first iteration runs eagerly (it sizes every buffer and sets the
    // kernels' attributes); with graphs on, the rest replay it as one CUDA
    // graph (~130 launches per iteration), the host convergence check every 8.
    // The sync-free triangular solves number their ready flags per solve on
    // the host, so SSOR / IC(0) keep the eager loop.
    // Opt-in (PMMF_B200_CG_GRAPH=1): measured on config 5, the replay gains
    // ~2% per iteration at 1024^2 and loses at 256^2 (gpurun_out/r02t).
    const char* ge = std::getenv("PMMF_B200_CG_GRAPH");
    const bool graph_ok = (!pc || pc->kind == PMMF_PRECOND_PMMF || pc->kind == PMMF_PRECOND_JACOBI) && ge &&
                          ge[0] == '1';
    int it = 0;
    if (cfg->max_iter >= 1) {
      iteration();
      it = 1;
    }
    cudaGraphExec_t exec = nullptr;
    if (graph_ok && it < cfg->max_iter) {
      cudaGraph_t graph = nullptr;
      PMMF_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      const int64_t launches0 = launch_counter().load();
      iteration();
      const int64_t per_iter = launch_counter().load() - launches0;
      PMMF_CUDA(cudaStreamEndCapture(s, &graph));
      PMMF_CUDA(cudaGraphInstantiate(&exec, graph, 0));
      cudaGraphDestroy(graph);
      launch_counter().fetch_sub(per_iter, std::memory_order_relaxed);  // counted per replay below
      while (it < cfg->max_iter) {
        const int k = std::min(8 - (it % 8 == 0 ? 0 : it % 8), cfg->max_iter - it);
        for (int q = 0; q < k; ++q) {
          PMMF_CUDA(cudaGraphLaunch(exec, s));
          launch_counter().fetch_add(per_iter, std::memory_order_relaxed);
        }
        it += k;
        if (all_done()) break;
      }
      cudaGraphExecDestroy(exec);
    } else {
      while (it < cfg->max_iter) {
        if (it % 8 == 0 && all_done()) break;
        iteration();
        ++it;
      }
    }
    std::vector<int32_t> hi = diters.to_host(nr), hc = dconv.to_host(nr), hbk = dbrk.to_host(nr);
    std::vector<double> ht = trace.to_host(static_cast<int64_t>(nr) * stride);
    for (int r = 0; r < nr; ++r) {
      if (bn[r] == 0.0) continue;
      iterations[r] = hi[r];
      converged[r] = hc[r];
      breakdown[r] = hbk[r];
      for (int i = 1; i < stride; ++i) residuals[static_cast<int64_t>(r) * stride + i] = ht[static_cast<int64_t>(r) * stride + i];
    }
    *wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - start).count();

}

}  // namespace pmmf_b200

using namespace pmmf_b200;

extern "C" {

int pmmf_b200_operator_create(void* result, double zero_threshold, void** op, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!result || !op) fail(PMMF_INVALID_ARGUMENT, "operator_create: null argument");
    auto o = std::make_unique<Operator>();
    o->thr = zero_threshold;
    o->build(*static_cast<Result*>(result));
    *op = o.release();
  });
}

int pmmf_b200_operator_apply(void* opv, int32_t mode, int64_t nrhs, const double* in, double* out, int32_t on_device,
                             char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    auto* o = static_cast<Operator*>(opv);
    if (mode < 0 || mode > 2) fail(PMMF_INVALID_ARGUMENT, "MmfOperator::apply: bad mode");
    if (nrhs < 1) return;
    PMMF_CUDA(cudaSetDevice(o->device));
    cudaStream_t s = o->s;
    const int64_t m = o->n * nrhs;
    DBuf<double> a(m, s), b(m, s);
    if (on_device)
      PMMF_CUDA(cudaMemcpyAsync(a.get(), in, sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
    else
      a.upload(in, m);
    to_index_major(a.get(), b.get(), o->n, static_cast<int>(nrhs), s);
    o->apply_dev(mode, static_cast<int>(nrhs), b.get(), s);
    to_rhs_major(b.get(), a.get(), o->n, static_cast<int>(nrhs), s);
    if (on_device)
      PMMF_CUDA(cudaMemcpyAsync(out, a.get(), sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
    else
      a.download(out, m);
    PMMF_CUDA(cudaStreamSynchronize(s));
  });
}

int pmmf_b200_operator_apply_sharded(void* opv, void* commv, int32_t mode, int64_t nrhs, const double* in,
                                     double* out, int32_t on_device, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    auto* o = static_cast<Operator*>(opv);
    const auto* C = static_cast<const Comm*>(commv);
    if (!o || !C) fail(PMMF_INVALID_ARGUMENT, "MmfOperator::apply (sharded): null argument");
    if (mode < 0 || mode > 2) fail(PMMF_INVALID_ARGUMENT, "MmfOperator::apply: bad mode");
    if (C->device != o->device) fail(PMMF_INVALID_ARGUMENT, "MmfOperator::apply (sharded): communicator on another device");
    if (nrhs < 1) return;
    PMMF_CUDA(cudaSetDevice(o->device));
    cudaStream_t s = o->s;
    const int64_t m = o->n * nrhs;
    DBuf<double> a(m, s), b(m, s);
    if (on_device)
      PMMF_CUDA(cudaMemcpyAsync(a.get(), in, sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
    else
      a.upload(in, m);
    to_index_major(a.get(), b.get(), o->n, static_cast<int>(nrhs), s);
    o->apply_dev_sharded(mode, static_cast<int>(nrhs), b.get(), s, *C);
    to_rhs_major(b.get(), a.get(), o->n, static_cast<int>(nrhs), s);
    if (on_device)
      PMMF_CUDA(cudaMemcpyAsync(out, a.get(), sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
    else
      a.download(out, m);
    PMMF_CUDA(cudaStreamSynchronize(s));
  });
}

// ||A - Q^T H Q||_F, dense (residual_frobenius with ResidualMethod::dense,
// transform_ops.hpp:225-237): Q^T H Q e_j for batches of unit vectors
// through the operator's forward apply (reconstruct_dense,
// transform_ops.hpp:175-213, by the apply's level order instead of the
// reference's rotation-by-rotation order: equal up to rounding), minus the
// dense input, squared and summed per batch by a fixed-shape reduction.
int pmmf_b200_residual_frobenius(void* result, const pmmf_b200_coo* a, int32_t method, int64_t cap, double* out,
                                 char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!result || !a || !out) fail(PMMF_INVALID_ARGUMENT, "residual_frobenius: null argument");
    const Result& f = *static_cast<Result*>(result);
    if (method == 0) {  // ResidualMethod::accumulated
      *out = std::sqrt(f.residual_sq);
      return;
    }
    if (method != 1) fail(PMMF_INVALID_ARGUMENT, "residual_frobenius: bad method");
    const int64_t n = f.n;
    if (n > cap) fail(PMMF_NUMERIC, "reconstruct_dense: dimension exceeds cap");
    if (a->n != n) fail(PMMF_INVALID_ARGUMENT, "residual_frobenius: matrix dimension differs");
    PMMF_CUDA(cudaSetDevice(a->device));
    Operator o;
    o.thr = 0.0;
    o.build(f);
    cudaStream_t s = o.s;
    // dense A, row-major (duplicates summed)
    DBuf<double> A(std::max<int64_t>(n * n, 1), s);
    A.zero();
    if (a->nnz > 0) {
      DBuf<int64_t> r, c;
      DBuf<double> v;
      const int64_t* pr = a->rows;
      const int64_t* pc = a->cols;
      const double* pv = a->vals;
      if (!a->on_device) {
        r.alloc(a->nnz, s);
        c.alloc(a->nnz, s);
        v.alloc(a->nnz, s);
        r.upload(a->rows, a->nnz);
        c.upload(a->cols, a->nnz);
        v.upload(a->vals, a->nnz);
        pr = r.get();
        pc = c.get();
        pv = v.get();
      }
      DBuf<int> bad(1, s);
      bad.zero();
      PMMF_LAUNCH(k_dense_scatter_coo, blocks_for(a->nnz, kThreads), kThreads, 0, s, a->nnz, n, pr, pc, pv, A.get(),
                  bad.get());
      if (bad.to_host(1)[0]) fail(PMMF_OUT_OF_RANGE, "residual_frobenius: index out of range");
    }
    const int nb = static_cast<int>(std::min<int64_t>(n, 256));
    DBuf<double> V(n * nb, s), part(1024, s);
    double total = 0.0;
    for (int64_t j0 = 0; j0 < n; j0 += nb) {
      const int cnt = static_cast<int>(std::min<int64_t>(nb, n - j0));
      PMMF_LAUNCH(k_unit_block, blocks_for(n * cnt, kThreads), kThreads, 0, s, n, cnt, j0, V.get());
      o.apply_dev(PMMF_APPLY_FORWARD, cnt, V.get(), s);
      PMMF_LAUNCH(k_diff_sq, 1024, kThreads, kThreads * sizeof(double), s, n, cnt, j0, A.get(), V.get(), part.get());
      const std::vector<double> h = part.to_host(1024);
      for (double x : h) total += x;
    }
    *out = std::sqrt(total);
  });
}

int pmmf_b200_operator_zeroed_negatives(void* op, int64_t* out) {
  *out = static_cast<Operator*>(op)->neg;
  return PMMF_OK;
}

void pmmf_b200_operator_free(void* op) { delete static_cast<Operator*>(op); }

int pmmf_b200_solve(const pmmf_b200_coo* a, void* opv, const pmmf_b200_solve_config* cfg, int32_t* iterations,
                    int32_t* converged, int32_t* breakdown, double* residuals, double* wall_ms, char* err,
                    size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!a || !cfg) fail(PMMF_INVALID_ARGUMENT, "solve: null argument");
    std::unique_ptr<SplitPrecond> pc;
    if (opv) pc = precond_from_operator(opv);
    run_cg(a, pc.get(), cfg, iterations, converged, breakdown, residuals, wall_ms);
  });
}

}  // extern "C"
