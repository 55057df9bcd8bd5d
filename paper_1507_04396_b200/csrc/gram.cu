// gram.cu — per-cluster Gram matrices G_u = A[:,B_u]^T A[:,B_u]
// (blocked_matrix.hpp:238-254) and diagonal blocks D_u = A[B_u,B_u]
// (:257-266) as dense column-major c_u x c_u tiles.
//
// Bitwise order: G[a][b] is the sequential sum over
// the rows of the stage numbering of A[r][a]*A[r][b].  The batch's entries
// are re-sorted once by (cluster, row) -- one stable LSD radix sort on a
// 32-bit key, columns staying ascending inside a run -- every CSC entry
// learns the row-run that holds its row inside its own cluster, and then a
// warp owns output column a: it walks column a's entries in row order and,
// per entry, adds the products with its row-run into G[:,a] — lanes on
// distinct b, rows strictly in order.  Work is sum_r deg_u(r)^2, the
// reference's own product count.
#include <cub/cub.cuh>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>

#include "engine.cuh"

namespace pmmf_b200 {

namespace {

constexpr int kThreads = 256;

// (cluster, row)-major view of a cluster batch: key = (cluster index in the
// batch) << rb | row, payload = entry index; ecol = column of every entry.
template <typename KeyT>
__global__ void k_entry_rows(i64 e0, const i64* __restrict__ ptr, i64 col0, i64 ncols,
                             const int32_t* __restrict__ row, const int32_t* __restrict__ col_seg, int rb,
                             KeyT* __restrict__ key, int32_t* __restrict__ idx, int32_t* __restrict__ ecol) {
  const i64 w = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= ncols) return;
  const i64 J = col0 + w;
  const KeyT hi = static_cast<KeyT>(col_seg[w]) << rb;
  for (i64 e = ptr[J] + lane; e < ptr[J + 1]; e += 32) {
    key[e - e0] = hi | static_cast<KeyT>(row[e]);
    idx[e - e0] = static_cast<int32_t>(e - e0);
    ecol[e - e0] = static_cast<int32_t>(J);
  }
}

// Runs of equal (cluster, row) keys in the sorted order: the head stamps
// [lo, hi) on every member, indexed by its original entry.
template <typename KeyT>
__global__ void k_key_runs(i64 ne, const KeyT* __restrict__ keys, const int32_t* __restrict__ idx,
                           int32_t* __restrict__ run_lo, int32_t* __restrict__ run_hi) {
  const i64 p = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (p >= ne) return;
  const KeyT k = keys[p];
  if (p > 0 && keys[p - 1] == k) return;
  i64 q = p + 1;
  while (q < ne && keys[q] == k) ++q;
  for (i64 t = p; t < q; ++t) {
    run_lo[idx[t]] = static_cast<int32_t>(p);
    run_hi[idx[t]] = static_cast<int32_t>(q);
  }
}

// Run entries in sorted order: column (stage id) and value.
__global__ void k_csr_fill(i64 ne, const int32_t* __restrict__ idx, const int32_t* __restrict__ ecol,
                           const double* __restrict__ val_base, int32_t* __restrict__ csr_col,
                           double* __restrict__ csr_val) {
  const i64 p = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (p >= ne) return;
  const int32_t e = idx[p];
  csr_col[p] = ecol[e];
  csr_val[p] = val_base[e];
}

// Owner-column accumulation into the dense tile.
__global__ void k_gram_owner(i64 col0, i64 ncols, i64 e0, const i64* __restrict__ ptr,
                             const double* __restrict__ val, const int32_t* __restrict__ run_lo,
                             const int32_t* __restrict__ run_hi, const int32_t* __restrict__ csr_col,
                             const double* __restrict__ csr_val, const int32_t* __restrict__ col_cluster_off,
                             const int64_t* __restrict__ col_tile, const int32_t* __restrict__ col_c,
                             double* __restrict__ G) {
  const i64 w = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= ncols) return;
  const i64 J = col0 + w;
  const int32_t cbase = col_cluster_off[w];
  const i64 a = J - cbase;
  const i64 c = col_c[w];
  double* Gcol = G + col_tile[w] + a * c;
  for (i64 e = ptr[J]; e < ptr[J + 1]; ++e) {
    const double va = val[e];
    const int32_t lo = run_lo[e - e0], hi = run_hi[e - e0];
    for (int32_t q = lo + lane; q < hi; q += 32) {
      const int32_t b = csr_col[q] - cbase;
      Gcol[b] = dadd(Gcol[b], dmul(va, csr_val[q]));
    }
    __syncwarp();
  }
}

// Products of an owner column (sum of its rows' run lengths): the sort key of
// the heaviest-first column order below.
__global__ void k_owner_cost(i64 col0, i64 ncols, i64 e0, const i64* __restrict__ ptr,
                             const int32_t* __restrict__ run_lo, const int32_t* __restrict__ run_hi,
                             int32_t* __restrict__ cost, int32_t* __restrict__ idx) {
  const i64 w = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= ncols) return;
  const i64 J = col0 + w;
  i64 c = 0;
  for (i64 e = ptr[J] + lane; e < ptr[J + 1]; e += 32) c += run_hi[e - e0] - run_lo[e - e0];
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) {
    cost[w] = static_cast<int32_t>(c < 0x7fffffff ? c : 0x7fffffff);
    idx[w] = static_cast<int32_t>(w);
  }
}

// Software-pipelined k_gram_owner (same sums in the same order).  The plain
// kernel pays three dependent global round trips per row of the owner column
// (run bounds -> run entries -> accumulator), ~31 rows in a row on config 4.
// Here a warp loads the (value, run) records of 32 rows at once, and while row
// t is accumulated the run entries of row t+2 are being loaded and the
// accumulator sectors of row t+1 are being prefetched (kPf = 1: into L1,
// 2: into L2), so a row costs one cache-hit read-modify-write.
template <int kPf>
__global__ void k_gram_owner_pipe(i64 col0, i64 ncols, i64 e0, const i64* __restrict__ ptr,
                                  const double* __restrict__ val, const int32_t* __restrict__ run_lo,
                                  const int32_t* __restrict__ run_hi, const int32_t* __restrict__ csr_col,
                                  const double* __restrict__ csr_val, const int32_t* __restrict__ col_cluster_off,
                                  const int64_t* __restrict__ col_tile, const int32_t* __restrict__ col_c,
                                  double* __restrict__ G, const int32_t* __restrict__ order) {
  const i64 w0 = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w0 >= ncols) return;
  // optional heaviest-first column order (ncu: achieved occupancy 32% of a
  // possible 62% in column order); measured slower, off by default
  const i64 w = order ? order[w0] : w0;
  const i64 J = col0 + w;
  const int32_t cbase = col_cluster_off[w];
  const i64 a = J - cbase;
  const i64 c = col_c[w];
  double* Gcol = G + col_tile[w] + a * c;
  const i64 end = ptr[J + 1];
  for (i64 base = ptr[J]; base < end; base += 32) {
    const int n = static_cast<int>(end - base < 32 ? end - base : 32);
    double va_l = 0.0;
    int32_t lo_l = 0, hi_l = 0;
    if (lane < n) {
      va_l = val[base + lane];
      lo_l = run_lo[base + lane - e0];
      hi_l = run_hi[base + lane - e0];
    }
    // stage A: the first 32 run entries of row x (b < 0: none for this lane)
    auto load_run = [&](int x, int32_t& b, double& pv, int32_t& lo, int32_t& hi) {
      lo = __shfl_sync(0xffffffffu, lo_l, x & 31);
      hi = __shfl_sync(0xffffffffu, hi_l, x & 31);
      b = -1;
      pv = 0.0;
      if (x < n && lo + lane < hi) {
        b = csr_col[lo + lane] - cbase;
        pv = csr_val[lo + lane];
      }
    };
    auto prefetch = [&](int32_t b) {
      if (kPf == 1 && b >= 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(Gcol + b));
      if (kPf == 2 && b >= 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(Gcol + b));
    };
    int32_t b0, b1, b2 = -1, lo0, hi0, lo1, hi1, lo2 = 0, hi2 = 0;
    double pv0, pv1, pv2 = 0.0;
    load_run(0, b0, pv0, lo0, hi0);
    load_run(1, b1, pv1, lo1, hi1);
    prefetch(b0);
    for (int t = 0; t < n; ++t) {
      if (t + 2 < n) load_run(t + 2, b2, pv2, lo2, hi2);
      prefetch(b1);
      const double va = __shfl_sync(0xffffffffu, va_l, t);
      if (b0 >= 0) Gcol[b0] = dadd(Gcol[b0], dmul(va, pv0));
      for (int32_t q = lo0 + 32 + lane; q < hi0; q += 32) {  // rows shared by more than 32 columns
        const int32_t b = csr_col[q] - cbase;
        Gcol[b] = dadd(Gcol[b], dmul(va, csr_val[q]));
      }
      __syncwarp();
      b0 = b1;
      pv0 = pv1;
      lo0 = lo1;
      hi0 = hi1;
      b1 = b2;
      pv1 = pv2;
      lo1 = lo2;
      hi1 = hi2;
      b2 = -1;
    }
  }
}

__global__ void k_run_total(i64 ne, const int32_t* __restrict__ lo, const int32_t* __restrict__ hi,
                            unsigned long long* __restrict__ tot) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  unsigned long long v = i < ne ? static_cast<unsigned long long>(hi[i] - lo[i]) : 0ull;
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(tot, v);
}

// D[r][a] = D[a][r] = A[r][a] for the upper triangle r <= a of block (u,u).
__global__ void k_diag_block(i64 col0, i64 ncols, const i64* __restrict__ ptr, const int32_t* __restrict__ row,
                             const double* __restrict__ val, const int32_t* __restrict__ col_cluster_off,
                             const int64_t* __restrict__ col_tile, const int32_t* __restrict__ col_c,
                             double* __restrict__ D) {
  const i64 w = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= ncols) return;
  const i64 J = col0 + w;
  const i64 off = col_cluster_off[w], a = J - off, c = col_c[w];
  double* T = D + col_tile[w];
  for (i64 e = ptr[J] + lane; e < ptr[J + 1]; e += 32) {
    const i64 r = static_cast<i64>(row[e]) - off;
    if (r < 0 || r > a) continue;
    T[a * c + r] = val[e];
    T[r * c + a] = val[e];
  }
}

// ------------------------------------------------------------ dense path
// A cluster whose columns are well filled is summed as a dense SYRK: its
// columns are scattered into a zero-filled column-major panel (ld = N, rows
// in stage order) and every output G[a][b] is accumulated by one thread
// over the rows strictly in ascending order with separately rounded
// products and sums -- the reference's sequence with exact-zero products
// inserted for rows where one side is absent.  0 + p = p, s + (+-0) = s for
// s != 0, so the value is the reference's up to the sign of an exact zero,
// which nothing downstream observes.

__global__ void k_panel_scatter(i64 col0, i64 ncols, i64 N, const i64* __restrict__ ptr,
                                const int32_t* __restrict__ row, const double* __restrict__ val,
                                double* __restrict__ panel) {
  const i64 w = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= ncols) return;
  double* P = panel + w * N;
  const i64 J = col0 + w;
  for (i64 e = ptr[J] + lane; e < ptr[J + 1]; e += 32) P[row[e]] = val[e];
}

struct DenseTile {
  int64_t pcol;   // panel column of the cluster's first member
  int64_t gtile;  // tile offset of the cluster in G
  int32_t c;      // cluster size
  int32_t bi, bj; // output tile (bi <= bj)
};

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool pred) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int n = pred ? 8 : 0;  // src-size 0: zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// 256 threads, tile BM = 16*TM outputs square, KC rows per smem stage,
// two-stage cp.async pipeline.  Thread (ty, tx) owns rows a in
// {ty*4 + 64*h + i} and columns b in {tx*4 + 64*h + j} (TM = 8) or
// {ty*4 + i} x {tx*4 + j} (TM = 4).
template <int TM>
__global__ void __launch_bounds__(256) k_syrk_seq(const DenseTile* __restrict__ tiles, i64 N,
                                                  const double* __restrict__ panel, double* __restrict__ G) {
  constexpr int BM = 16 * TM;
  constexpr int KC = 16;
  constexpr int LD = BM + 4;  // 32-byte aligned rows
  constexpr int PER = KC * BM / 256;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                 // [2][KC][LD]
  double* Bs = smem + 2 * KC * LD;   // [2][KC][LD]
  const DenseTile t = tiles[blockIdx.x];
  const int c = t.c;
  const int a0 = t.bi * BM, b0 = t.bj * BM;
  const double* Pa = panel + (t.pcol + a0) * N;
  const double* Pb = panel + (t.pcol + b0) * N;
  const int tid = threadIdx.x;
  const int ty = tid >> 4, tx = tid & 15;

  auto load = [&](int st, i64 r0) {
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int idx = tid + 256 * i;
      const int k = idx & (KC - 1), x = idx / KC;
      const bool rk = r0 + k < N;
      const bool pa = rk && a0 + x < c, pb = rk && b0 + x < c;
      cp_async8(As + (st * KC + k) * LD + x, pa ? Pa + static_cast<i64>(x) * N + r0 + k : Pa, pa);
      cp_async8(Bs + (st * KC + k) * LD + x, pb ? Pb + static_cast<i64>(x) * N + r0 + k : Pb, pb);
    }
    cp_async_commit();
  };

  double acc[TM][TM];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TM; ++j) acc[i][j] = 0.0;

  const i64 nchunks = (N + KC - 1) / KC;
  load(0, 0);
  for (i64 ch = 0; ch < nchunks; ++ch) {
    const int st = static_cast<int>(ch & 1);
    if (ch + 1 < nchunks) {
      load(st ^ 1, (ch + 1) * KC);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* Ak = As + st * KC * LD;
    const double* Bk = Bs + st * KC * LD;
#pragma unroll 4
    for (int k = 0; k < KC; ++k) {
      double av[TM], bv[TM];
#pragma unroll
      for (int h = 0; h < TM / 4; ++h) {
        const double2 x0 = *reinterpret_cast<const double2*>(Ak + k * LD + ty * 4 + 64 * h);
        const double2 x1 = *reinterpret_cast<const double2*>(Ak + k * LD + ty * 4 + 64 * h + 2);
        const double2 y0 = *reinterpret_cast<const double2*>(Bk + k * LD + tx * 4 + 64 * h);
        const double2 y1 = *reinterpret_cast<const double2*>(Bk + k * LD + tx * 4 + 64 * h + 2);
        av[4 * h] = x0.x; av[4 * h + 1] = x0.y; av[4 * h + 2] = x1.x; av[4 * h + 3] = x1.y;
        bv[4 * h] = y0.x; bv[4 * h + 1] = y0.y; bv[4 * h + 2] = y1.x; bv[4 * h + 3] = y1.y;
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TM; ++j) acc[i][j] = dadd(acc[i][j], dmul(av[i], bv[j]));
    }
    __syncthreads();
  }
  double* Gt = G + t.gtile;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int a = a0 + ty * 4 + 64 * (i / 4) + (i & 3);
    if (a >= c) continue;
#pragma unroll
    for (int j = 0; j < TM; ++j) {
      const int b = b0 + tx * 4 + 64 * (j / 4) + (j & 3);
      if (b >= c) continue;
      Gt[static_cast<i64>(b) * c + a] = acc[i][j];
      if (t.bi != t.bj) Gt[static_cast<i64>(a) * c + b] = acc[i][j];
    }
  }
}

// ---------------------------------------------------------------- DMMA path
// Opt-in (pmmf_b200_set_dense_gram(1)): the dense Gram on the FP64 tensor
// cores.  mma.sync m8n8k4 f64 (DMMA) accumulates each 4-row k-step with its
// own rounding, so G differs from the reference's sequential sum in the
// last bits and a pivot whose score margin is that small can flip (the
// near-tie clause of SURVEY.md §8(c)); the bitwise SIMT SYRK stays the
// default.  Operands are staged by TMA (cp.async.bulk.tensor, 128-byte
// swizzle, boxes of 16 rows x 128 panel columns) into a 3-stage mbarrier
// pipeline; 128 x 128 output tile per CTA, 8 warps of 32 x 64, 32 DMMA per
// warp per k-step.
constexpr int kDmT = 128;          // output tile edge
constexpr int kDmKC = 32;          // k rows per pipeline stage
constexpr int kDmStages = 3;
constexpr int kDmBox = 16 * kDmT * 8;              // bytes of one 16 x 128 box
constexpr int kDmStageBytes = 4 * kDmBox;          // A (2 boxes) + B (2 boxes)
constexpr int kDmSmem = kDmStages * kDmStageBytes + 1024;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
// Element (panel column x in [0,128), row k in [0,16)) of a 128B-swizzled box.
__device__ __forceinline__ const double* box_at(const char* box, int x, int k) {
  return reinterpret_cast<const double*>(box + x * 128 + ((((k >> 1) ^ (x & 7))) << 4) + ((k & 1) << 3));
}

__global__ void __launch_bounds__(256, 1) k_syrk_dmma(const __grid_constant__ CUtensorMap map,
                                                      const DenseTile* __restrict__ tiles, i64 N,
                                                      double* __restrict__ G) {
  extern __shared__ __align__(1024) char dm_smem[];
  char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(dm_smem) + 1023) & ~uintptr_t{1023});
  __shared__ __align__(8) uint64_t full[kDmStages];
  const DenseTile t = tiles[blockIdx.x];
  const int c = t.c;
  const int a0 = t.bi * kDmT, b0 = t.bj * kDmT;
  const int ca = static_cast<int>(t.pcol) + a0, cb = static_cast<int>(t.pcol) + b0;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, tg = lane & 3;
  const int wa = (w >> 1) * 32, wb = (w & 1) * 64;
  const int nch = static_cast<int>((N + kDmKC - 1) / kDmKC);
  if (tid == 0) {
    for (int i = 0; i < kDmStages; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int ch) {
    const int st = ch % kDmStages;
    char* sb = base + st * kDmStageBytes;
    mbar_expect(&full[st], kDmStageBytes);
    const int k0 = ch * kDmKC;
    tma_load_2d(sb, &map, k0, ca, &full[st]);
    tma_load_2d(sb + kDmBox, &map, k0 + 16, ca, &full[st]);
    tma_load_2d(sb + 2 * kDmBox, &map, k0, cb, &full[st]);
    tma_load_2d(sb + 3 * kDmBox, &map, k0 + 16, cb, &full[st]);
  };
  if (tid == 0)
    for (int ch = 0; ch < kDmStages - 1 && ch < nch; ++ch) issue(ch);
  double acc[4][8][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int ch = 0; ch < nch; ++ch) {
    const int st = ch % kDmStages;
    if (tid == 0 && ch + kDmStages - 1 < nch) issue(ch + kDmStages - 1);
    mbar_wait(&full[st], static_cast<uint32_t>((ch / kDmStages) & 1));
    const char* sb = base + st * kDmStageBytes;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const char* Ab = sb + h * kDmBox;
      const char* Bb = sb + (2 + h) * kDmBox;
#pragma unroll
      for (int ks = 0; ks < 16; ks += 4) {
        double av[4], bv[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = *box_at(Ab, wa + 8 * i + g, ks + tg);
#pragma unroll
        for (int j = 0; j < 8; ++j) bv[j] = *box_at(Bb, wb + 8 * j + g, ks + tg);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) dmma(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
      }
    }
    __syncthreads();  // the stage is refilled next iteration
  }
  double* Gt = G + t.gtile;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int a = a0 + wa + 8 * i + g;
    if (a >= c) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int b = b0 + wb + 8 * j + 2 * tg + q;
        if (b >= c) continue;
        Gt[static_cast<i64>(b) * c + a] = acc[i][j][q];
        if (t.bi != t.bj) Gt[static_cast<i64>(a) * c + b] = acc[i][j][q];
      }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    (void)cudaGetLastError();
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  if (!fn) fail(PMMF_CUDA, "gram (DMMA): cuTensorMapEncodeTiled unavailable");
  return fn;
}

std::atomic<int>& dense_gram_mode() {
  static std::atomic<int> m{[] {
    const char* e = std::getenv("PMMF_B200_GRAM_DMMA");
    return e && e[0] == '1' ? 1 : 0;
  }()};
  return m;
}

// Per-column cluster info from the cluster offsets (block per cluster): was
// built column by column on the host and uploaded from pageable memory
// (16 MB at n = 2^20, every stage).
__global__ void k_col_info(const i64* __restrict__ off, const i64* __restrict__ tile, i64 col0, i64 tile0,
                           int32_t* __restrict__ cco, int32_t* __restrict__ cc, int64_t* __restrict__ ct) {
  const i64 b = off[blockIdx.x], e = off[blockIdx.x + 1];
  for (i64 J = b + threadIdx.x; J < e; J += blockDim.x) {
    cco[J - col0] = static_cast<int32_t>(b);
    cc[J - col0] = static_cast<int32_t>(e - b);
    ct[J - col0] = tile[blockIdx.x] - tile0;
  }
}
__global__ void k_col_seg(const i64* __restrict__ off, i64 col0, int32_t* __restrict__ seg) {
  const i64 b = off[blockIdx.x], e = off[blockIdx.x + 1];
  for (i64 J = b + threadIdx.x; J < e; J += blockDim.x) seg[J - col0] = static_cast<int32_t>(blockIdx.x);
}
__global__ void k_ptr_at(i64 n, const i64* __restrict__ ptr, const i64* __restrict__ cols, i64* __restrict__ out) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = ptr[cols[i]];
}

// Sparse path over the contiguous clusters [v0, v1) (column arrays indexed
// from the batch's first column, offset by cbase).
void gram_sparse(const Csc& a, const std::vector<i64>& off, i64 v0, i64 v1, i64 e0, i64 ne, const int32_t* dcco,
                 const int64_t* dct, const int32_t* dcc, double* G, cudaStream_t s) {
  const i64 col0 = off[v0], ncols = off[v1] - off[v0];
  if (ncols <= 0 || ne <= 0) return;
  if (ne >= (i64{1} << 31)) fail(PMMF_INTERNAL, "gram: cluster batch exceeds 2^31 entries");
  // One stable radix sort on (cluster index in the run, row) keeps the
  // columns ascending inside a run; a run is a row's entries inside the
  // owner column's own cluster.
  const i64 N = a.N;
  const i64 nseg = v1 - v0;
  const int rb = std::max(1, bits_for(std::max<i64>(N - 1, 1)));
  const int sb = std::max(1, bits_for(std::max<i64>(nseg - 1, 1)));
  DBuf<int32_t> dseg(ncols, s);
  {
    DBuf<i64> doff(nseg + 1, s);
    doff.upload(off.data() + v0, nseg + 1);
    PMMF_LAUNCH(k_col_seg, static_cast<unsigned>(nseg), 256, 0, s, doff.get(), col0, dseg.get());
  }
  DBuf<int32_t> idx(ne, s), idx2(ne, s), ecol(ne, s), run_lo(ne, s), run_hi(ne, s);
  auto sorted_runs = [&](auto zero_key) {
    using KeyT = decltype(zero_key);
    DBuf<KeyT> key(ne, s), key2(ne, s);
    PMMF_LAUNCH(k_entry_rows<KeyT>, blocks_for(ncols * 32, kThreads), kThreads, 0, s, e0, a.ptr.get(), col0, ncols,
                a.row.get(), dseg.get(), rb, key.get(), idx.get(), ecol.get());
    size_t tmp = 0;
    PMMF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key.get(), key2.get(), idx.get(), idx2.get(),
                                              static_cast<int64_t>(ne), 0, rb + sb, s));
    DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
    PMMF_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, key.get(), key2.get(), idx.get(), idx2.get(),
                                              static_cast<int64_t>(ne), 0, rb + sb, s));
    PMMF_LAUNCH(k_key_runs<KeyT>, blocks_for(ne, kThreads), kThreads, 0, s, ne, key2.get(), idx2.get(), run_lo.get(),
                run_hi.get());
  };
  if (rb + sb <= 32)
    sorted_runs(uint32_t{0});
  else
    sorted_runs(uint64_t{0});
  idx.release();
  DBuf<int32_t> csr_col(ne, s);
  DBuf<double> csr_val(ne, s);
  PMMF_LAUNCH(k_csr_fill, blocks_for(ne, kThreads), kThreads, 0, s, ne, idx2.get(), ecol.get(), a.val.get() + e0,
              csr_col.get(), csr_val.get());
  idx2.release();
  ecol.release();
  // Resident warps bound the live accumulator columns (c doubles each) that
  // compete for L2; unused dynamic shared memory caps the warps per SM
  // (PMMF_B200_GRAM_OWNER_SMEM bytes per 256-thread block, tuning hook).
  static const int owner_smem = [] {
    const char* e = std::getenv("PMMF_B200_GRAM_OWNER_SMEM");
    return e ? std::atoi(e) : 0;
  }();
  if (owner_smem > 48 * 1024)
    PMMF_CUDA(cudaFuncSetAttribute(k_gram_owner, cudaFuncAttributeMaxDynamicSharedMemorySize, owner_smem));
  // PMMF_B200_GRAM_PIPE: 0 = plain kernel, 1 / 2 = pipelined with L1 / L2 accumulator prefetch, 3 = pipelined, none
  // (read per call; measured, config 4 gram phase: 0: 150, 1: 143.8, 2: 146.1, 3: 142.9 ms)
  const char* pipe_env = std::getenv("PMMF_B200_GRAM_PIPE");
  const int pipe = pipe_env ? std::atoi(pipe_env) : 3;
#define PMMF_OWNER_ARGS                                                                                              \
  col0, ncols, e0, a.ptr.get(), a.val.get(), run_lo.get(), run_hi.get(), csr_col.get(), csr_val.get(), dcco, dct, dcc, G
  DBuf<int32_t> order;
  const char* lpt_env = std::getenv("PMMF_B200_GRAM_LPT");
  // opt-in (PMMF_B200_GRAM_LPT=1), measured and rejected: gram phase 145 -> 153-159 ms on config 4
  if (pipe != 0 && lpt_env && lpt_env[0] == '1' && ncols > 4096) {
    DBuf<int32_t> cost(ncols, s), cost2(ncols, s), idx0(ncols, s);
    order.alloc(ncols, s);
    PMMF_LAUNCH(k_owner_cost, blocks_for(ncols * 32, kThreads), kThreads, 0, s, col0, ncols, e0, a.ptr.get(),
                run_lo.get(), run_hi.get(), cost.get(), idx0.get());
    size_t tmp = 0;
    PMMF_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, cost.get(), cost2.get(), idx0.get(), order.get(),
                                                        static_cast<int64_t>(ncols), 0, 31, s));
    DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
    PMMF_CUDA(cub::DeviceRadixSort::SortPairsDescending(t.get(), tmp, cost.get(), cost2.get(), idx0.get(), order.get(),
                                                        static_cast<int64_t>(ncols), 0, 31, s));
  }
  const int32_t* dord = order.get();
  if (pipe == 1)
    PMMF_LAUNCH(k_gram_owner_pipe<1>, blocks_for(ncols * 32, kThreads), kThreads, owner_smem, s, PMMF_OWNER_ARGS, dord);
  else if (pipe == 2)
    PMMF_LAUNCH(k_gram_owner_pipe<2>, blocks_for(ncols * 32, kThreads), kThreads, owner_smem, s, PMMF_OWNER_ARGS, dord);
  else if (pipe == 3)
    PMMF_LAUNCH(k_gram_owner_pipe<0>, blocks_for(ncols * 32, kThreads), kThreads, owner_smem, s, PMMF_OWNER_ARGS, dord);
  else
    PMMF_LAUNCH(k_gram_owner, blocks_for(ncols * 32, kThreads), kThreads, owner_smem, s, PMMF_OWNER_ARGS);
#undef PMMF_OWNER_ARGS
  if (trace_enabled()) {  // products = sum over entries of their row-run length (the reference's count)
    DBuf<unsigned long long> tot(1, s);
    tot.zero();
    PMMF_LAUNCH(k_run_total, blocks_for(ne, kThreads), kThreads, 0, s, ne, run_lo.get(), run_hi.get(), tot.get());
    std::fprintf(stderr, "[pmmf]   gram sparse: %lld columns, %lld entries, %llu products\n",
                 static_cast<long long>(ncols), static_cast<long long>(ne), tot.to_host(1)[0]);
  }
}

// Dense path over clusters [v0, v1): one panel, one SYRK launch.
void gram_dense(const Csc& a, const std::vector<i64>& off, i64 v0, i64 v1, i64 u0, const std::vector<i64>& tile_off,
                double* G, cudaStream_t s) {
  const i64 col0 = off[v0], ncols = off[v1] - off[v0], N = a.N;
  if (ncols <= 0) return;
  i64 max_c = 0;
  for (i64 u = v0; u < v1; ++u) max_c = std::max(max_c, off[u + 1] - off[u]);
  // TM = 8 (128-wide tiles) unless that leaves the SMs short of work.
  auto count_tiles = [&](int bm) {
    i64 n = 0;
    for (i64 u = v0; u < v1; ++u) {
      const i64 nt = (off[u + 1] - off[u] + bm - 1) / bm;
      n += nt * (nt + 1) / 2;
    }
    return n;
  };
  const bool dmma = dense_gram_mode().load() == 1;
  const int tm = dmma ? 8 : (count_tiles(128) >= 2 * 148 ? 8 : 4);
  const int bm = dmma ? kDmT : 16 * tm;
  std::vector<DenseTile> tl;
  for (i64 u = v0; u < v1; ++u) {
    const i64 c = off[u + 1] - off[u];
    const i64 nt = (c + bm - 1) / bm;
    for (i64 bj = 0; bj < nt; ++bj)
      for (i64 bi = 0; bi <= bj; ++bi)
        tl.push_back({off[u] - col0, tile_off[u] - tile_off[u0], static_cast<int32_t>(c), static_cast<int32_t>(bi),
                      static_cast<int32_t>(bj)});
  }
  if (tl.empty()) return;
  // panel leading dimension: even for TMA (16-byte global strides)
  const i64 ld = dmma ? (N + 1) / 2 * 2 : N;
  DBuf<double> panel(ncols * ld, s);
  panel.zero();
  PMMF_LAUNCH(k_panel_scatter, blocks_for(ncols * 32, kThreads), kThreads, 0, s, col0, ncols, ld, a.ptr.get(),
              a.row.get(), a.val.get(), panel.get());
  DBuf<DenseTile> dtl(static_cast<i64>(tl.size()), s);
  PMMF_CUDA(cudaMemcpyAsync(dtl.get(), tl.data(), sizeof(DenseTile) * tl.size(), cudaMemcpyHostToDevice, s));
  const size_t smem = sizeof(double) * 2 * 2 * 16 * (bm + 4);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (prof_enabled()) {
    e0 = EventPool::get().take();
    e1 = EventPool::get().take();
    cudaEventRecord(e0, s);
  }
  if (dmma) {
    CUtensorMap map{};
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(ncols)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
    const cuuint32_t box[2] = {16, static_cast<cuuint32_t>(kDmT)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = tensor_map_encoder()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, panel.get(), dims, strides, box,
                                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(PMMF_CUDA, "gram (DMMA): tensor map encode failed (" + std::to_string(r) + ")");
    PMMF_CUDA(cudaFuncSetAttribute(k_syrk_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize, kDmSmem));
    PMMF_LAUNCH(k_syrk_dmma, static_cast<unsigned>(tl.size()), 256, kDmSmem, s, map, dtl.get(), N, G);
  } else if (tm == 8) {
    PMMF_CUDA(cudaFuncSetAttribute(k_syrk_seq<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    PMMF_LAUNCH(k_syrk_seq<8>, static_cast<unsigned>(tl.size()), 256, smem, s, dtl.get(), N, panel.get(), G);
  } else {
    PMMF_CUDA(cudaFuncSetAttribute(k_syrk_seq<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    PMMF_LAUNCH(k_syrk_seq<4>, static_cast<unsigned>(tl.size()), 256, smem, s, dtl.get(), N, panel.get(), G);
  }
  double flops = 0.0;  // R_u * c_u * (c_u + 1) per cluster
  for (i64 u = v0; u < v1; ++u) {
    const double c = static_cast<double>(off[u + 1] - off[u]);
    flops += static_cast<double>(N) * c * (c + 1.0);
  }
  if (e0) {
    cudaEventRecord(e1, s);
    PMMF_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    EventPool::get().give(e0);
    EventPool::get().give(e1);
    prof_add_n(dmma ? "gram_dmma" : "gram_dense", 1, ms, flops);
  }
  if (trace_enabled()) {
    PMMF_CUDA(cudaStreamSynchronize(s));
    std::fprintf(stderr, "[pmmf]   gram dense%s: %lld clusters, %lld columns x %lld rows, %zu tiles of %d, %.3g flop\n",
                 dmma ? " (DMMA)" : "", static_cast<long long>(v1 - v0), static_cast<long long>(ncols),
                 static_cast<long long>(N), tl.size(), bm, flops);
  }
}

// Dense-vs-sparse choice: the sparse path costs ~ sum_r deg_u(r)^2 >= nnz_u^2 / N
// scattered read-modify-writes, the dense one N c (c+1) / 2 register MACs.
double dense_ratio() {
  if (const char* e = std::getenv("PMMF_B200_GRAM_DENSE_RATIO")) return std::atof(e);  // test hook / tuning
  return 32.0;
}

}  // namespace

void gram_tiles(const Csc& a, const std::vector<i64>& off, i64 u0, i64 u1, const std::vector<i64>& tile_off,
                double* G, double* D, cudaStream_t s) {
  const i64 col0 = off[u0], ncols = off[u1] - off[u0];
  if (ncols <= 0) return;
  const i64 nb = u1 - u0;
  // per-column cluster info
  DBuf<int32_t> dcco(ncols, s), dcc(ncols, s);
  DBuf<int64_t> dct(ncols, s);
  // entry offsets at the cluster boundaries
  std::vector<i64> eptr;
  {
    DBuf<i64> cols(nb + 1, s), at(nb + 1, s), dtile(nb + 1, s);
    cols.upload(off.data() + u0, nb + 1);
    dtile.upload(tile_off.data() + u0, nb + 1);
    PMMF_LAUNCH(k_col_info, static_cast<unsigned>(nb), 256, 0, s, cols.get(), dtile.get(), col0, tile_off[u0],
                dcco.get(), dcc.get(), dct.get());
    PMMF_LAUNCH(k_ptr_at, blocks_for(nb + 1, kThreads), kThreads, 0, s, nb + 1, a.ptr.get(), cols.get(), at.get());
    eptr = at.to_host(nb + 1);
  }
  PMMF_LAUNCH(k_diag_block, blocks_for(ncols * 32, kThreads), kThreads, 0, s, col0, ncols, a.ptr.get(), a.row.get(),
              a.val.get(), dcco.get(), dct.get(), dcc.get(), D);
  const double ratio = dense_ratio();
  const double N = static_cast<double>(a.N);
  // dense panels are bounded by a share of free memory
  const i64 panel_cap = std::max<i64>(i64{1} << 24, available_bytes() / 4 / 8);
  auto is_dense = [&](i64 u) {
    const double c = static_cast<double>(off[u + 1] - off[u]);
    const double nz = static_cast<double>(eptr[u + 1 - u0] - eptr[u - u0]);
    return ratio > 0.0 && nz > 0.0 && N * c * (c + 1.0) * 0.5 <= ratio * nz * nz / N &&
           static_cast<i64>(c) * a.N <= panel_cap;
  };
  i64 v0 = u0;
  while (v0 < u1) {
    const bool dense = is_dense(v0);
    i64 v1 = v0 + 1;
    if (dense) {
      i64 cols = off[v0 + 1] - off[v0];
      while (v1 < u1 && is_dense(v1) && (cols + off[v1 + 1] - off[v1]) * a.N <= panel_cap) {
        cols += off[v1 + 1] - off[v1];
        ++v1;
      }
      gram_dense(a, off, v0, v1, u0, tile_off, G, s);
    } else {
      while (v1 < u1 && !is_dense(v1)) ++v1;
      const i64 w = off[v0] - col0;
      const i64 ne = eptr[v1 - u0] - eptr[v0 - u0];
      gram_sparse(a, off, v0, v1, eptr[v0 - u0], ne, dcco.get() + w, dct.get() + w, dcc.get() + w, G, s);
    }
    v0 = v1;
  }
}

}  // namespace pmmf_b200

extern "C" int pmmf_b200_set_dense_gram(int32_t mode) {
  if (mode != 0 && mode != 1) return PMMF_INVALID_ARGUMENT;
  pmmf_b200::dense_gram_mode().store(mode);
  return PMMF_OK;
}
extern "C" int32_t pmmf_b200_get_dense_gram(void) { return pmmf_b200::dense_gram_mode().load(); }

