// cluster.cu — randomized anchor clustering (clustering.hpp:85-225) with the
// data-parallel parts on the device:
//   * column norms, summed per block row of the PRE-reblock matrix then over
//     blocks (blocked_matrix.hpp:203-209),
//   * normalized scores |<A_j,A_a>| / (|A_j| |A_a|) of every pool column
//     against the m anchors and the strict-> argmax with ties to the lowest
//     anchor (clustering.hpp:62-83, P3/P4).  A warp owns a column; the
//     anchors are inverted into a row -> (anchor, value) index, so the work
//     is sum over the column's entries of the anchors sharing that row
//     (a sparse 2-hop gather), and each (column, anchor) dot keeps the
//     reference's two-level summation order exactly.
// The control flow that consumes the RNG stream (anchor draws, round-robin,
// undersize repair, oversize recursion) runs on the host, as in the
// reference, over device-computed scores.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <memory>
#include <numeric>
#include <type_traits>
#include <unordered_map>

#include "engine.cuh"
#include "rng.cuh"
#include "shard.cuh"

namespace pmmf_b200 {

namespace {

constexpr int kThreads = 256;

// Two-level column norm, warp per column (columns listed by stage id):
// lanes load 32 consecutive entries (coalesced) and square them; every lane
// then replays the reference's sequential order (inner sum per block row,
// flushed into the outer sum at block changes) through shuffles.
__global__ void k_norms(i64 P, const int32_t* __restrict__ cols, const i64* __restrict__ ptr,
                        const int32_t* __restrict__ row, const double* __restrict__ val,
                        const int32_t* __restrict__ blk, double* __restrict__ norm, i64 long_len, i64 c0,
                        i64 c1) {
  const i64 p = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= P) return;
  const int32_t j = cols[p];
  if (j < c0 || j >= c1) return;               // another rank's column
  if (ptr[j + 1] - ptr[j] > long_len) return;  // k_norms_long
  double s = 0.0, inner = 0.0;
  int32_t cur = -1;
  const i64 e1 = ptr[j + 1];
  for (i64 e0 = ptr[j]; e0 < e1; e0 += 32) {
    const i64 e = e0 + lane;
    double sq = 0.0;
    int32_t b = -1;
    if (e < e1) {
      const double v = val[e];
      sq = dmul(v, v);
      b = blk[row[e]];
    }
    const int n = e1 - e0 < 32 ? static_cast<int>(e1 - e0) : 32;
    for (int i = 0; i < n; ++i) {
      const int32_t bi = __shfl_sync(0xffffffffu, b, i);
      const double si = __shfl_sync(0xffffffffu, sq, i);
      if (bi != cur) {
        if (cur >= 0) s = dadd(s, inner);
        inner = 0.0;
        cur = bi;
      }
      inner = dadd(inner, si);
    }
  }
  if (cur >= 0) s = dadd(s, inner);
  if (lane == 0) norm[p] = sqrt(s);
}

// Long columns (hub columns after a stage's fill-in: up to ~n/2 entries,
// which one warp would sum serially for milliseconds): a CTA per column,
// thread per pre-reblock block.  Block u's part of the column is the row
// range [off[u], off[u+1]) (blocks are contiguous stage-id ranges, rows are
// ascending), summed sequentially by its thread; the column norm then adds
// the block sums in block order, empty blocks included, exactly as
// column_norm_sq does (blocked_matrix.hpp:203-209, sparse.hpp:99-103).
constexpr int kNormLongThreads = 256;
__global__ void __launch_bounds__(kNormLongThreads) k_norms_long(const int32_t* __restrict__ list,
                                                                 const int32_t* __restrict__ cols,
                                                                 const i64* __restrict__ ptr,
                                                                 const int32_t* __restrict__ row,
                                                                 const double* __restrict__ val, const i64* __restrict__ off,
                                                                 i64 nblk, double* __restrict__ part,
                                                                 double* __restrict__ norm) {
  const i64 p = list[blockIdx.x];
  const int32_t j = cols[p];
  const i64 e0 = ptr[j], e1 = ptr[j + 1];
  double* my = part + static_cast<i64>(blockIdx.x) * nblk;
  auto lb = [&](i64 key) {
    i64 lo = e0, hi = e1;
    while (lo < hi) {
      const i64 mid = (lo + hi) >> 1;
      if (row[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  for (i64 u = threadIdx.x; u < nblk; u += blockDim.x) {
    const i64 b = lb(off[u]), e = lb(off[u + 1]);
    double s = 0.0;
    for (i64 x = b; x < e; ++x) {
      const double v = val[x];
      s = dadd(s, dmul(v, v));
    }
    my[u] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (i64 u = 0; u < nblk; ++u) s = dadd(s, my[u]);
    norm[p] = sqrt(s);
  }
}

__global__ void k_long_flags(i64 P, const int32_t* __restrict__ cols, const i64* __restrict__ ptr, i64 long_len,
                             uint8_t* __restrict__ flag) {
  const i64 p = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (p < P) flag[p] = ptr[cols[p] + 1] - ptr[cols[p]] > long_len ? 1 : 0;
}

// Row -> anchor index: count, then scatter (order inside a row is free:
// each anchor appears at most once per row).
__global__ void k_anchor_count(int m, const int32_t* __restrict__ anchors, const i64* __restrict__ ptr,
                               const int32_t* __restrict__ row, int32_t* __restrict__ cnt) {
  const int a = blockIdx.x;
  const int32_t j = anchors[a];
  for (i64 e = ptr[j] + threadIdx.x; e < ptr[j + 1]; e += blockDim.x) atomicAdd(&cnt[row[e]], 1);
}
__global__ void k_anchor_scatter(int m, const int32_t* __restrict__ anchors, const i64* __restrict__ ptr,
                                 const int32_t* __restrict__ row, const double* __restrict__ val,
                                 const i64* __restrict__ rptr, int32_t* __restrict__ cursor,
                                 int32_t* __restrict__ ent_a, double* __restrict__ ent_v) {
  const int a = blockIdx.x;
  const int32_t j = anchors[a];
  for (i64 e = ptr[j] + threadIdx.x; e < ptr[j + 1]; e += blockDim.x) {
    const int32_t r = row[e];
    const i64 pos = rptr[r] + atomicAdd(&cursor[r], 1);
    ent_a[pos] = a;
    ent_v[pos] = val[e];
  }
}
__global__ void k_widen(i64 N, const int32_t* __restrict__ in, i64* __restrict__ out) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < N) out[i] = in[i];
  if (i == N) out[i] = 0;
}

struct ScoreArgs {
  i64 P;
  const int32_t* cols;    // pool columns (stage ids)
  const double* cnorm;    // their norms
  int m;
  const double* anorm;    // anchor norms
  const int32_t* self;    // stage id -> anchor position or -1 (assignment mode)
  const i64* ptr;
  const int32_t* row;
  const double* val;
  const int32_t* blk;
  const i64* arptr;       // row -> anchor entries
  const int32_t* ent_a;
  const double* ent_v;
  int32_t* assign;        // assignment mode: best anchor or -1
  double* rows;           // rows mode: P x m scores (nullptr in assignment mode)
  double* g_scratch;      // per-warp state when shared memory is too small
  unsigned long long* stats;  // trace: {hit rows, anchor entries} (nullable)
  long long* col_cycles;      // trace: cycles per pool column (nullable)
  long long* warp_cycles;     // trace: busy cycles per warp (nullable)
  const int32_t* anchors;     // anchor stage ids (dense path)
  const int32_t* list;        // pool positions handled by k_score, heaviest first
  i64 nlist;
  unsigned long long* next;   // work counter over list
};

__device__ __forceinline__ bool better(double s, int a, double bs, int ba) {
  return s > bs || (s == bs && a < ba);
}

constexpr int kPrefetch = 8;  // anchor entries of a hit row staged in shared memory

// Per-warp state: block partial p[m], total t[m], last block seen last[m],
// then the prefetch buffers (16-byte aligned).
// ... plus the list of anchors the current column touched (m int32) and its
// length, so a column's epilogue costs its touched anchors, not m.
// Narrow layout (anchors and pre-reblock blocks < 32768, every BASELINE
// config): 16-bit last-block, touched-list and staged anchor indices, 12.5 KB
// instead of 15.0 KB per warp at m = 512 -> 17 instead of 14 resident warps per
// SM for a kernel whose issue rate is set by its resident warps (ncu: 3.5
// active and 0.32 eligible warps per scheduler).
__host__ __device__ constexpr size_t score_pf_off(int m, bool narrow) {
  return (static_cast<size_t>(m) * (narrow ? 20 : 24) + 4 + 15) / 16 * 16;
}
__host__ __device__ constexpr size_t score_stride(int m, bool narrow) {
  return score_pf_off(m, narrow) + 32 * kPrefetch * (narrow ? 10 : 12) + 32;
}

// Warps loop over pool columns.  For every chunk of 32 entries of the
// column, each lane stages the first kPrefetch (anchor, value) pairs of its
// row in shared memory; then the rows with anchors are replayed in row
// order (the reference's summation order per anchor), lanes spread over the
// row's anchors, updating the two-level accumulators of distinct anchors.
// kSmem: per-warp state in shared memory (else in a global scratch slot,
// for anchor counts whose state exceeds shared memory).
template <bool kSmem, bool kNarrow>
__global__ void k_score(ScoreArgs A, int warps_per_block) {
  using last_t = std::conditional_t<kNarrow, int16_t, int32_t>;
  using idx_t = std::conditional_t<kNarrow, uint16_t, int32_t>;
  extern __shared__ __align__(16) unsigned char smem[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const i64 gwarp = blockIdx.x * static_cast<i64>(warps_per_block) + wib;
  const int m = A.m;
  const size_t stride = score_stride(m, kNarrow);
  unsigned char* base;
  if constexpr (kSmem)
    base = smem + stride * wib;
  else
    base = reinterpret_cast<unsigned char*>(A.g_scratch) + stride * static_cast<size_t>(gwarp);
  double* p = reinterpret_cast<double*>(base);
  double* t = p + m;
  last_t* last = reinterpret_cast<last_t*>(t + m);
  idx_t* touched = reinterpret_cast<idx_t*>(last + m);
  int32_t* ntouched = reinterpret_cast<int32_t*>(touched + m);
  double* pf_v = reinterpret_cast<double*>(base + score_pf_off(m, kNarrow));
  idx_t* pf_a = reinterpret_cast<idx_t*>(pf_v + 32 * kPrefetch);
  uint8_t* slotmap = reinterpret_cast<uint8_t*>(pf_a + 32 * kPrefetch);  // window slot -> row lane
  for (int a = lane; a < m; a += 32) {
    p[a] = 0.0;
    t[a] = 0.0;
    last[a] = static_cast<last_t>(-1);
  }
  if (lane == 0) *ntouched = 0;
  __syncwarp();
  long long busy = 0;
  unsigned long long st_rows = 0, st_ent = 0;  // trace counters, flushed once per warp
  for (;;) {  // columns fetched dynamically, heaviest first
    i64 idx = 0;
    if (lane == 0) idx = static_cast<i64>(atomicAdd(A.next, 1ull));
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx >= A.nlist) break;
    const i64 w = A.list[idx];
    const long long c_start = A.col_cycles ? clock64() : 0;
    const int32_t j = A.cols[w];
    if (A.rows == nullptr && A.self[j] >= 0) {
      if (lane == 0) A.assign[w] = A.self[j];
      if (A.col_cycles && lane == 0) A.col_cycles[w] = 0;
      continue;
    }
    const i64 e0 = A.ptr[j], e1 = A.ptr[j + 1];
    // chunk loads are software-pipelined one chunk ahead
    double nv = 0.0;
    int32_t nb = 0;
    i64 nbeg = 0, ncnt = 0;
    {
      const i64 e = e0 + lane;
      if (e < e1) {
        const int32_t r = A.row[e];
        nv = A.val[e];
        nb = A.blk[r];
        nbeg = A.arptr[r];
        ncnt = A.arptr[r + 1] - nbeg;
      }
    }
    for (i64 base_e = e0; base_e < e1; base_e += 32) {
      const double v = nv;
      const int32_t b = nb;
      const i64 beg = nbeg, cnt = ncnt;
      {
        const i64 e = base_e + 32 + lane;
        nv = 0.0;
        nb = 0;
        nbeg = 0;
        ncnt = 0;
        if (e < e1) {
          const int32_t r = A.row[e];
          nv = A.val[e];
          nb = A.blk[r];
          nbeg = A.arptr[r];
          ncnt = A.arptr[r + 1] - nbeg;
        }
      }
      if (cnt <= kPrefetch) {
#pragma unroll
        for (int k = 0; k < kPrefetch; ++k)
          if (k < cnt) {
            pf_a[lane * kPrefetch + k] = static_cast<idx_t>(A.ent_a[beg + k]);
            pf_v[lane * kPrefetch + k] = A.ent_v[beg + k];
          }
      }
      __syncwarp();
      // Update of anchor a by row (value vr, block br) with anchor value av:
      // the block partial p restarts at 0.0 on a new block row and the
      // finished partial is flushed into the total t (two-level order, P3).
      auto update = [&](int32_t a, double vr, int32_t br, double av) {
        const double prod = dmul(vr, av);
        const int32_t la = last[a];
        const double pa = p[a], ta = t[a];
        const bool same = la == br;
        if (la < 0) touched[atomicAdd(ntouched, 1)] = static_cast<idx_t>(a);
        t[a] = (same || la < 0) ? ta : dadd(ta, pa);
        p[a] = dadd(same ? pa : 0.0, prod);
        last[a] = static_cast<last_t>(br);
      };
      // Light rows (<= kPrefetch anchors, staged in shared memory) are packed
      // into windows of <= 32 (row, anchor) slots in row order; an anchor
      // shared by several rows of a window is updated one row per round,
      // in row order.  Heavy rows are processed alone.
      const unsigned hit_mask = __ballot_sync(0xffffffffu, cnt > 0);
      const unsigned heavy_mask = __ballot_sync(0xffffffffu, cnt > kPrefetch);
      const int c32 = cnt > 0 ? static_cast<int>(cnt < 32 ? cnt : 32) : 0;
      int incl = c32;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
      }
      const int excl = incl - c32;
      unsigned hits = hit_mask;
      while (hits) {
        const int s0 = __ffs(hits) - 1;
        if ((heavy_mask >> s0) & 1u) {
          hits &= hits - 1;
          const double vs = __shfl_sync(0xffffffffu, v, s0);
          const int32_t bs = __shfl_sync(0xffffffffu, b, s0);
          const i64 bg = __shfl_sync(0xffffffffu, beg, s0);
          const i64 n = __shfl_sync(0xffffffffu, cnt, s0);
          st_rows += 1;
          st_ent += static_cast<unsigned long long>(n);
          if (n <= 32) {  // one slot per lane
            if (lane < n) update(A.ent_a[bg + lane], vs, bs, A.ent_v[bg + lane]);
          } else {
            // hub row: issue all of a 256-entry batch's loads before any update
            constexpr int kB = 8;
            for (i64 q0 = 0; q0 < n; q0 += 32 * kB) {
              int32_t ra[kB];
              double rv[kB];
#pragma unroll
              for (int k = 0; k < kB; ++k) {
                const i64 q = q0 + k * 32 + lane;
                ra[k] = q < n ? A.ent_a[bg + q] : 0;
                rv[k] = q < n ? A.ent_v[bg + q] : 0.0;
              }
#pragma unroll
              for (int k = 0; k < kB; ++k)
                if (q0 + k * 32 + lane < n) update(ra[k], vs, bs, rv[k]);
            }
          }
          __syncwarp();
          continue;
        }
        const int base = __shfl_sync(0xffffffffu, excl, s0);
        const unsigned later_heavy = heavy_mask & (0xffffffffu << s0);
        const int stop = later_heavy ? __ffs(later_heavy) - 1 : 32;
        const bool fits = ((hits >> lane) & 1u) && lane < stop && incl - base <= 32;
        const unsigned win = __ballot_sync(0xffffffffu, fits);
        const int total = __shfl_sync(0xffffffffu, incl, 31 - __clz(win)) - base;
        if (fits)
          for (int k = 0; k < c32; ++k) slotmap[excl - base + k] = static_cast<uint8_t>(lane);
        __syncwarp();
        const bool on = lane < total;
        const int src = on ? slotmap[lane] : lane;
        const int k = lane - (__shfl_sync(0xffffffffu, excl, src) - base);
        const double vs = __shfl_sync(0xffffffffu, v, src);
        const int32_t bs = __shfl_sync(0xffffffffu, b, src);
        const int32_t a = on ? static_cast<int32_t>(pf_a[src * kPrefetch + k]) : -1 - lane;
        const double av = on ? pf_v[src * kPrefetch + k] : 0.0;
        const unsigned grp = __match_any_sync(0xffffffffu, a);
        const int rk = __popc(grp & ((1u << lane) - 1u));
        const int rounds = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(__popc(grp))));
        for (int r = 0; r < rounds; ++r) {
          if (on && rk == r) update(a, vs, bs, av);
          __syncwarp();
        }
        st_rows += static_cast<unsigned long long>(__popc(win));
        st_ent += static_cast<unsigned long long>(total);
        hits &= ~win;
      }
    }
    __syncwarp();
    const double nj = A.cnorm[w];
    double best = 0.0;
    int ba = 0x7fffffff;
    const int nt = *ntouched;  // untouched anchors: dot 0, score 0
    for (int i = lane; i < nt; i += 32) {
      const int a = touched[i];
      const double dot = dadd(t[a], p[a]);
      const double na = A.anorm[a];
      double sc = 0.0;
      if (nj > 0.0 && na > 0.0) sc = fabs(dot) / dmul(nj, na);
      if (A.rows) A.rows[static_cast<size_t>(w) * m + a] = sc;
      if (sc > 0.0 && better(sc, a, best, ba)) {
        best = sc;
        ba = a;
      }
      p[a] = 0.0;  // reset for the next column
      t[a] = 0.0;
      last[a] = static_cast<last_t>(-1);
    }
    __syncwarp();
    if (lane == 0) *ntouched = 0;
    for (int o = 16; o; o >>= 1) {
      const double os = __shfl_xor_sync(0xffffffffu, best, o);
      const int oa = __shfl_xor_sync(0xffffffffu, ba, o);
      if (better(os, oa, best, ba)) {
        best = os;
        ba = oa;
      }
    }
    if (lane == 0 && A.rows == nullptr) A.assign[w] = best > 0.0 ? ba : -1;
    __syncwarp();
    if (A.col_cycles && lane == 0) {
      const long long c = clock64() - c_start;
      A.col_cycles[w] = c;
      busy += c;
    }
  }
  if (A.warp_cycles && lane == 0) A.warp_cycles[gwarp] = busy;
  if (A.stats && lane == 0) {
    atomicAdd(&A.stats[0], st_rows);
    atomicAdd(&A.stats[1], st_ent);
  }
}

// Serial work of a pool column in k_score (self-assigned anchors cost
// nothing).  Sort key for the work list.
__global__ void k_col_cost(i64 P, const int32_t* __restrict__ cols, const int32_t* __restrict__ self, bool rows_mode,
                           const i64* __restrict__ ptr, const int32_t* __restrict__ row, const int32_t* __restrict__ cnt,
                           int32_t* __restrict__ key, int32_t* __restrict__ idx) {
  const i64 p = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= P) return;
  const int32_t j = cols[p];
  i64 c = 0;  // warp steps: one per hit row plus one per 16 anchor entries
  if (rows_mode || self[j] < 0)
    for (i64 e = ptr[j] + lane; e < ptr[j + 1]; e += 32) {
      const int32_t n = cnt[row[e]];
      c += n > 0 ? 1 + n / 16 : 0;
    }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) {
    key[p] = static_cast<int32_t>(c < 0x7fffffff ? c : 0x7fffffff);
    idx[p] = static_cast<int32_t>(p);
  }
}
__global__ void k_count_above(i64 n, const int32_t* __restrict__ key, int32_t thr, int32_t* __restrict__ out) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  // keys sorted descending: the boundary is where key crosses thr
  if (i < n && key[i] > thr && (i + 1 == n || key[i + 1] <= thr)) *out = static_cast<int32_t>(i + 1);
}

// Dense path for the heaviest pool columns (hub columns hit by most rows).
// A batch of D such columns is scattered into X (row-major N x D, zero
// elsewhere); then a warp owns (anchor a, 32 consecutive batch columns) and
// walks a's entries once in row order: the row, value and block are
// warp-uniform, X[r, d..d+31] is one coalesced load, and each lane keeps the
// two-level (block partial, total) sum of its column.  Rows outside a
// column give zero products; adding a zero never changes a non-zero partial
// and only the sign of a zero dot can differ, which |dot| removes, so the
// scores equal the sparse path's bit for bit.
__global__ void k_dense_scatter(const int32_t* __restrict__ dcols, const int32_t* __restrict__ cols,
                                const i64* __restrict__ ptr, const int32_t* __restrict__ row,
                                const double* __restrict__ val, int D, bool clear, double* __restrict__ X) {
  const int d = blockIdx.x;
  const int32_t j = cols[dcols[d]];
  for (i64 e = ptr[j] + threadIdx.x; e < ptr[j + 1]; e += blockDim.x)
    X[static_cast<i64>(row[e]) * D + d] = clear ? 0.0 : val[e];
}

__global__ void __launch_bounds__(256) k_score_spmm(ScoreArgs A, const int32_t* __restrict__ aorder, int G,
                                                    const int32_t* __restrict__ dcols, int Dcur, int D,
                                                    const double* __restrict__ X, double* __restrict__ S) {
  const i64 gw = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= static_cast<i64>(A.m) * G) return;
  const int a = aorder[gw / G];
  const int d = static_cast<int>(gw % G) * 32 + lane;
  const int32_t aj = A.anchors[a];
  const i64 f0 = A.ptr[aj], f1 = A.ptr[aj + 1];
  const double* xc = X + (d < D ? d : D - 1);
  double tot = 0.0, inner = 0.0;
  int32_t cur = -1;
  // 32 entries per round: all 32 X loads are issued before the sum chain
  for (i64 fb = f0; fb < f1; fb += 32) {
    const i64 f = fb + lane;
    int32_t r = 0, b = -1;
    double v = 0.0;
    if (f < f1) {
      r = A.row[f];
      v = A.val[f];
      b = A.blk[r];
    }
    const int n = f1 - fb < 32 ? static_cast<int>(f1 - fb) : 32;
    double xv[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) xv[k] = xc[static_cast<i64>(__shfl_sync(0xffffffffu, r, k)) * D];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const double vk = __shfl_sync(0xffffffffu, v, k);
      const int32_t bk = __shfl_sync(0xffffffffu, b, k);
      if (k < n) {
        const double prod = dmul(xv[k], vk);
        if (bk != cur) {
          if (cur >= 0) tot = dadd(tot, inner);
          inner = 0.0;
          cur = bk;
        }
        inner = dadd(inner, prod);
      }
    }
  }
  if (d >= Dcur) return;
  const double dot = cur >= 0 ? dadd(tot, inner) : 0.0;
  const i64 w = dcols[d];
  const double nj = A.cnorm[w], na = A.anorm[a];
  const double sc = (nj > 0.0 && na > 0.0) ? fabs(dot) / dmul(nj, na) : 0.0;
  if (A.rows)
    A.rows[static_cast<size_t>(w) * A.m + a] = sc;
  else
    S[static_cast<i64>(d) * A.m + a] = sc;
}

// Strict argmax over the anchors of a dense batch column (ties: lowest anchor).
__global__ void k_dense_argmax(ScoreArgs A, const int32_t* __restrict__ dcols, int Dcur,
                               const double* __restrict__ S) {
  const i64 d = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (d >= Dcur) return;
  double best = 0.0;
  int ba = 0x7fffffff;
  for (int a = lane; a < A.m; a += 32) {
    const double sc = S[d * A.m + a];
    if (sc > 0.0 && better(sc, a, best, ba)) {
      best = sc;
      ba = a;
    }
  }
  for (int o = 16; o; o >>= 1) {
    const double os = __shfl_xor_sync(0xffffffffu, best, o);
    const int oa = __shfl_xor_sync(0xffffffffu, ba, o);
    if (better(os, oa, best, ba)) {
      best = os;
      ba = oa;
    }
  }
  if (lane == 0) A.assign[dcols[d]] = best > 0.0 ? ba : -1;
}

// ------------------------------------------------------------ GEMM path
// Dense problems (configs 1 and 3: every column full): the pool and anchor
// columns are scattered into zero-filled column-major panels (ld = N) and
// the P x m dot products are computed as a tiled SIMT GEMM.  Each thread
// keeps, per anchor, the reference's two-level sum (column_dot,
// blocked_matrix.hpp:193-201): a block partial summed over the rows of one
// pre-reblock block in ascending order, folded into the total when the
// block changes (the row chunk's blocks are CTA-uniform).  Inserted rows
// contribute exact-zero products: only the sign of a zero dot can differ,
// which |dot| removes, so the scores are the sparse path's bit for bit.
constexpr int kGemmKC = 32, kGemmTJ = 64, kGemmTA = 32;

__global__ void k_panel_cols(i64 n, const int32_t* __restrict__ cols, const i64* __restrict__ ptr,
                             const int32_t* __restrict__ row, const double* __restrict__ val, i64 N,
                             double* __restrict__ X) {
  const i64 w = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  const int32_t j = cols[w];
  double* x = X + w * N;
  for (i64 e = ptr[j] + lane; e < ptr[j + 1]; e += 32) x[row[e]] = val[e];
}

__global__ void __launch_bounds__(256) k_score_gemm(i64 N, int Pc, int m, const double* __restrict__ Xp,
                                                    const double* __restrict__ Xa, const int32_t* __restrict__ blk,
                                                    const double* __restrict__ pnorm,
                                                    const double* __restrict__ anorm, double* __restrict__ S) {
  constexpr int KC = kGemmKC, TJ = kGemmTJ, TA = kGemmTA, AT = TA / 4;
  __shared__ double ps[KC][TJ + 1];
  __shared__ double as[KC][TA + 1];
  __shared__ int32_t bs[KC];
  const int j0 = blockIdx.x * TJ, a0 = blockIdx.y * TA;
  const int tid = threadIdx.x, tj = tid % TJ, ag = tid / TJ;
  double inner[AT], tot[AT];
#pragma unroll
  for (int i = 0; i < AT; ++i) inner[i] = tot[i] = 0.0;
  int32_t cur = -1;
  for (i64 r0 = 0; r0 < N; r0 += KC) {
#pragma unroll
    for (int i = 0; i < KC * TJ / 256; ++i) {
      const int idx = tid + 256 * i, k = idx % KC, j = idx / KC;
      ps[k][j] = (j0 + j < Pc && r0 + k < N) ? Xp[static_cast<i64>(j0 + j) * N + r0 + k] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < KC * TA / 256; ++i) {
      const int idx = tid + 256 * i, k = idx % KC, a = idx / KC;
      as[k][a] = (a0 + a < m && r0 + k < N) ? Xa[static_cast<i64>(a0 + a) * N + r0 + k] : 0.0;
    }
    if (tid < KC) bs[tid] = r0 + tid < N ? blk[r0 + tid] : -1;
    __syncthreads();
    const int kn = N - r0 < KC ? static_cast<int>(N - r0) : KC;
    for (int k = 0; k < kn; ++k) {
      const int32_t b = bs[k];
      if (b != cur) {  // CTA-uniform
        if (cur >= 0) {
#pragma unroll
          for (int i = 0; i < AT; ++i) tot[i] = dadd(tot[i], inner[i]);
        }
#pragma unroll
        for (int i = 0; i < AT; ++i) inner[i] = 0.0;
        cur = b;
      }
      const double x = ps[k][tj];
#pragma unroll
      for (int i = 0; i < AT; ++i) inner[i] = dadd(inner[i], dmul(x, as[k][ag * AT + i]));
    }
    __syncthreads();
  }
  const int j = j0 + tj;
  if (j >= Pc) return;
  const double nj = pnorm[j];
#pragma unroll
  for (int i = 0; i < AT; ++i) {
    const int a = a0 + ag * AT + i;
    if (a >= m) continue;
    const double dot = cur >= 0 ? dadd(tot[i], inner[i]) : 0.0;
    const double na = anorm[a];
    S[static_cast<i64>(j) * m + a] = (nj > 0.0 && na > 0.0) ? fabs(dot) / dmul(nj, na) : 0.0;
  }
}

// Assignment from a P x m score table: self-assigned anchors keep their own
// position (clustering.hpp:118-122); else the strict argmax (ties: lowest).
__global__ void k_gemm_argmax(i64 Pc, int m, const int32_t* __restrict__ cols, const int32_t* __restrict__ self,
                              const double* __restrict__ S, int32_t* __restrict__ assign) {
  const i64 d = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (d >= Pc) return;
  const int32_t sf = self[cols[d]];
  double best = 0.0;
  int ba = 0x7fffffff;
  for (int a = lane; a < m; a += 32) {
    const double sc = S[d * m + a];
    if (sc > 0.0 && better(sc, a, best, ba)) {
      best = sc;
      ba = a;
    }
  }
  for (int o = 16; o; o >>= 1) {
    const double os = __shfl_xor_sync(0xffffffffu, best, o);
    const int oa = __shfl_xor_sync(0xffffffffu, ba, o);
    if (better(os, oa, best, ba)) {
      best = os;
      ba = oa;
    }
  }
  if (lane == 0) assign[d] = sf >= 0 ? sf : (best > 0.0 ? ba : -1);
}

__global__ void k_anchor_nnz(int m, const int32_t* __restrict__ anchors, const i64* __restrict__ ptr,
                             int32_t* __restrict__ nnz, int32_t* __restrict__ idx) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= m) return;
  const i64 c = ptr[anchors[a] + 1] - ptr[anchors[a]];
  nnz[a] = static_cast<int32_t>(c < 0x7fffffff ? c : 0x7fffffff);
  idx[a] = a;
}

struct Scorer {
  const Csc& a;
  const Numbering& nb;
  cudaStream_t s;
  int force_gemm = -1;         // >= 0: the GEMM / sparse choice made for the whole matrix
  DBuf<int32_t> self;  // stage id -> anchor pos (assignment mode)

  Scorer(const Csc& mat, const Numbering& numbering, cudaStream_t st) : a(mat), nb(numbering), s(st) {
    self.alloc(std::max<i64>(a.N, 1), s);
    self.fill_bytes(0xff);
  }

  // Scores of the P pool columns `dpool` (stage ids, device) against the m
  // `danch` (stage ids, ascending global; device).  Assignment mode writes
  // the best anchor or -1 per pool column to assign_out (device); rows mode
  // writes the full P x m score table to rows_out (device).
  void run(const int32_t* dpool, const double* dpn, i64 P, const int32_t* danch, const double* dan, int m,
           bool rows_mode, int32_t* assign_out, double* rows_out) {
    if (P == 0) return;
    const auto t_start = std::chrono::steady_clock::now();
    if (gemm_mode()) {
      run_gemm(P, m, dpool, dpn, danch, dan, rows_mode, assign_out, rows_out, t_start);
      return;
    }
    // row -> anchor index
    DBuf<int32_t> cnt(a.N + 1, s), cursor(a.N + 1, s);
    cnt.zero();
    cursor.zero();
    PMMF_LAUNCH(k_anchor_count, static_cast<unsigned>(m), 128, 0, s, m, danch, a.ptr.get(), a.row.get(), cnt.get());
    DBuf<i64> cnt64(a.N + 1, s), rptr(a.N + 1, s);
    PMMF_LAUNCH(k_widen, blocks_for(a.N + 1, kThreads), kThreads, 0, s, a.N, cnt.get(), cnt64.get());
    {
      size_t tmp = 0;
      PMMF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt64.get(), rptr.get(), static_cast<int64_t>(a.N + 1), s));
      DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
      PMMF_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, cnt64.get(), rptr.get(), static_cast<int64_t>(a.N + 1), s));
    }
    i64 total = 0;
    PMMF_CUDA(cudaMemcpyAsync(&total, rptr.get() + a.N, sizeof(i64), cudaMemcpyDeviceToHost, s));
    PMMF_CUDA(cudaStreamSynchronize(s));
    DBuf<int32_t> ent_a(std::max<i64>(total, 1), s);
    DBuf<double> ent_v(std::max<i64>(total, 1), s);
    PMMF_LAUNCH(k_anchor_scatter, static_cast<unsigned>(m), 128, 0, s, m, danch, a.ptr.get(), a.row.get(),
                a.val.get(), rptr.get(), cursor.get(), ent_a.get(), ent_v.get());
    if (!rows_mode) {
      std::vector<int32_t> pos(static_cast<size_t>(m));
      std::iota(pos.begin(), pos.end(), 0);
      // mark anchors (self-assignment, clustering.hpp:118-122)
      DBuf<int32_t> dpos(m, s);
      dpos.upload(pos);
      set_self(danch, dpos.get(), m, true);
    }
    // warps per block: most resident warps per SM under the shared-memory
    // limit (227 KB per SM, 1 KB reserved per block)
    const bool narrow = m <= 32767 && nb.clusters() <= 32767;
    const size_t stride = score_stride(m, narrow);
    int wpb = 0, best_w = 0;
    for (int w = 1; w <= 18; ++w) {  // 18 warps x 104 registers fit the register file of one block
      const size_t per_block = stride * static_cast<size_t>(w);
      if (per_block + 1024 > 227 * 1024) break;
      const int bps = std::min<int>(32, static_cast<int>((227 * 1024) / (per_block + 1024)));
      if (w * bps > best_w) {
        best_w = w * bps;
        wpb = w;
      }
    }
    const bool use_smem = wpb >= 1;
    if (!use_smem) wpb = 4;
    DBuf<double> scratch;
    if (!use_smem)  // one state slot per launched warp (persistent grid of 148 x 8 blocks)
      scratch.alloc(static_cast<i64>((stride * static_cast<size_t>(148 * 8 * wpb) + 7) / 8), s);
    int32_t* dassign = assign_out;
    if (rows_mode) PMMF_CUDA(cudaMemsetAsync(rows_out, 0, sizeof(double) * P * m, s));
    ScoreArgs args{P,           dpool,       dpn,              m,           dan,         self.get(),
                   a.ptr.get(), a.row.get(), a.val.get(),      nb.d_blk.get(), rptr.get(), ent_a.get(),
                   ent_v.get(), dassign, rows_mode ? rows_out : nullptr, scratch.get(), nullptr,
                   nullptr, nullptr, danch, nullptr, 0, nullptr};
    // Work list: pool positions by decreasing serial cost (rows hit); the
    // heaviest, above a share of the anchors' total size, take the dense path.
    DBuf<int32_t> key(P, s), key2(P, s), idx(P, s), list(P, s), nd_d(1, s);
    PMMF_LAUNCH(k_col_cost, blocks_for(P * 32, kThreads), kThreads, 0, s, P, dpool, self.get(), rows_mode,
                a.ptr.get(), a.row.get(), cnt.get(), key.get(), idx.get());
    {
      size_t tmp = 0;
      PMMF_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, key.get(), key2.get(), idx.get(), list.get(),
                                                          static_cast<int64_t>(P), 0, 32, s));
      DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
      PMMF_CUDA(cub::DeviceRadixSort::SortPairsDescending(t.get(), tmp, key.get(), key2.get(), idx.get(), list.get(),
                                                          static_cast<int64_t>(P), 0, 32, s));
    }
    double thr_d = std::max<double>(64.0, static_cast<double>(total) / 4.0);
    if (const char* e = std::getenv("PMMF_B200_DENSE_DIV")) {  // test hook: no floor, <= 0 disables
      const double div = std::atof(e);
      thr_d = div > 0.0 ? static_cast<double>(total) / div : 1e18;
    }
    const int32_t thr = static_cast<int32_t>(std::min<double>(0x7ffffffe, thr_d));
    nd_d.zero();
    PMMF_LAUNCH(k_count_above, blocks_for(P, kThreads), kThreads, 0, s, P, key2.get(), thr, nd_d.get());
    const i64 nd = nd_d.to_host(1)[0];
    DBuf<unsigned long long> next(1, s);
    next.zero();
    args.list = list.get() + nd;
    args.nlist = P - nd;
    args.next = next.get();
    const size_t smem = use_smem ? stride * static_cast<size_t>(wpb) : 0;
    if (smem > 48 * 1024)
      PMMF_CUDA(cudaFuncSetAttribute(narrow ? k_score<true, true> : k_score<true, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    // persistent grid: resident warps loop over the work list
    const i64 blocks = std::min<i64>((P + wpb - 1) / wpb, use_smem ? 148 * std::max(1, best_w / wpb) : 148 * 8);
    DBuf<unsigned long long> stats;
    DBuf<long long> ccyc, wcyc;
    const bool timing = trace_enabled() && std::getenv("PMMF_B200_SCORE_TIMING");
    if (trace_enabled()) {
      stats.alloc(2, s);
      stats.zero();
      args.stats = stats.get();
    }
    if (timing) {
      ccyc.alloc(P, s);
      ccyc.zero();
      wcyc.alloc(blocks * wpb, s);
      wcyc.zero();
      args.col_cycles = ccyc.get();
      args.warp_cycles = wcyc.get();
    }
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    if (timing)
      for (auto& e : ev) cudaEventCreate(&e);
    if (timing) cudaEventRecord(ev[0], s);
    int dense_D = 0, max_annz = 0;
    if (nd > 0) {
      // anchors by decreasing size (longest walks start first)
      DBuf<int32_t> ann(m, s), ann2(m, s), aidx(m, s), aorder(m, s);
      PMMF_LAUNCH(k_anchor_nnz, blocks_for(m, kThreads), kThreads, 0, s, m, danch, a.ptr.get(), ann.get(),
                  aidx.get());
      {
        size_t tmp = 0;
        PMMF_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, ann.get(), ann2.get(), aidx.get(),
                                                            aorder.get(), m, 0, 32, s));
        DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
        PMMF_CUDA(cub::DeviceRadixSort::SortPairsDescending(t.get(), tmp, ann.get(), ann2.get(), aidx.get(),
                                                            aorder.get(), m, 0, 32, s));
      }
      // batch width: X (N x D fp64) within a fifth of free memory, a multiple
      // of 32 (each batch re-walks every anchor: fewer, wider batches)
      const i64 budget = std::max<i64>(i64{1} << 30, available_bytes() / 5);
      const i64 dmax = std::max<i64>(32, budget / (8 * std::max<i64>(a.N, 1)) / 32 * 32);
      const int D = static_cast<int>(std::min<i64>(dmax, (nd + 31) / 32 * 32));
      const int G = D / 32;
      dense_D = D;
      if (timing) max_annz = ann2.to_host(1)[0];
      DBuf<double> X(static_cast<i64>(D) * a.N, s), S;
      X.zero();
      if (!rows_mode) S.alloc(static_cast<i64>(D) * m, s);
      for (i64 d0 = 0; d0 < nd; d0 += D) {
        const int Dcur = static_cast<int>(std::min<i64>(D, nd - d0));
        const int32_t* dcols = list.get() + d0;
        PMMF_LAUNCH(k_dense_scatter, static_cast<unsigned>(Dcur), 256, 0, s, dcols, dpool, a.ptr.get(),
                    a.row.get(), a.val.get(), D, false, X.get());
        PMMF_LAUNCH(k_score_spmm, blocks_for(static_cast<i64>(m) * G * 32, 256), 256, 0, s, args, aorder.get(), G,
                    dcols, Dcur, D, X.get(), S.get());
        if (!rows_mode)
          PMMF_LAUNCH(k_dense_argmax, blocks_for(static_cast<i64>(Dcur) * 32, kThreads), kThreads, 0, s, args, dcols,
                      Dcur, S.get());
        PMMF_LAUNCH(k_dense_scatter, static_cast<unsigned>(Dcur), 256, 0, s, dcols, dpool, a.ptr.get(),
                    a.row.get(), a.val.get(), D, true, X.get());
      }
    }
    if (timing) cudaEventRecord(ev[1], s);
    auto launch_sparse = [&] {
      if (args.nlist <= 0) return;
      if (use_smem && narrow)
        PMMF_LAUNCH((k_score<true, true>), static_cast<unsigned>(blocks), 32 * wpb, smem, s, args, wpb);
      else if (use_smem)
        PMMF_LAUNCH((k_score<true, false>), static_cast<unsigned>(blocks), 32 * wpb, smem, s, args, wpb);
      else if (narrow)
        PMMF_LAUNCH((k_score<false, true>), static_cast<unsigned>(blocks), 32 * wpb, 0, s, args, wpb);
      else
        PMMF_LAUNCH((k_score<false, false>), static_cast<unsigned>(blocks), 32 * wpb, 0, s, args, wpb);
    };
    launch_sparse();
    if (timing) cudaEventRecord(ev[2], s);
    if (trace_enabled()) {
      std::vector<unsigned long long> h = stats.to_host(2);
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
      std::fprintf(stderr, "[pmmf]   score: pool=%lld anchors=%d dense=%lld hit_rows=%llu anchor_entries=%llu %.2f ms\n",
                   static_cast<long long>(P), m, static_cast<long long>(nd), h[0], h[1], ms);
      if (timing) {
        std::vector<long long> cc = ccyc.to_host(P), wc = wcyc.to_host(blocks * wpb);
        std::vector<long long> dc;
        for (long long& c : cc)
          if (c < 0) {
            dc.push_back(-c);
            c = 0;
          }
        const double csum = std::accumulate(cc.begin(), cc.end(), 0.0);
        const double dsum = std::accumulate(dc.begin(), dc.end(), 0.0);
        std::sort(cc.begin(), cc.end(), std::greater<long long>());
        std::sort(dc.begin(), dc.end(), std::greater<long long>());
        const long long wmax = *std::max_element(wc.begin(), wc.end());
        float t1 = 0.f, t2 = 0.f;
        cudaEventElapsedTime(&t1, ev[0], ev[1]);
        cudaEventElapsedTime(&t2, ev[1], ev[2]);
        std::fprintf(stderr,
                     "[pmmf]     score: dense %.2f ms (thr %d, E_anchor %lld, max %d, D %d) sparse %.2f ms"
                     " (sum %.3g cyc, top %lld %lld %lld, warps %lld max %lld mean %.3g)\n",
                     t1, thr, static_cast<long long>(total), max_annz, dense_D, t2, csum, cc[0],
                     cc[std::min<i64>(1, P - 1)], cc[std::min<i64>(10, P - 1)], static_cast<long long>(blocks * wpb),
                     wmax, csum / static_cast<double>(blocks * wpb));
      }
      for (auto& e : ev)
        if (e) cudaEventDestroy(e);
    }
    if (!rows_mode) set_self(danch, danch, m, false);
  }

  void set_self(const int32_t* anchors, const int32_t* pos, int m, bool on);

  // Dense problems go through the GEMM path: at least a quarter of all
  // entries stored (PMMF_B200_SCORE_GEMM=1/0 forces it on/off for tests).
  bool gemm_mode() const {
    if (const char* e = std::getenv("PMMF_B200_SCORE_GEMM")) return std::atoi(e) != 0;
    if (force_gemm >= 0) return force_gemm != 0;
    const double N = static_cast<double>(a.N);
    return a.N > 0 && static_cast<double>(a.nnz) >= 0.25 * N * N;
  }

  void run_gemm(i64 P, int m, const int32_t* dpool, const double* dpn, const int32_t* danch, const double* dan,
                bool rows_mode, int32_t* assign_out, double* rows_out, std::chrono::steady_clock::time_point t_start) {
    const i64 N = a.N;
    if (!rows_mode) {  // mark anchors (self-assignment, clustering.hpp:118-122)
      std::vector<int32_t> pos(static_cast<size_t>(m));
      std::iota(pos.begin(), pos.end(), 0);
      DBuf<int32_t> dpos(m, s);
      dpos.upload(pos);
      set_self(danch, dpos.get(), m, true);
    }
    DBuf<double> Xa(static_cast<i64>(m) * N, s);
    Xa.zero();
    PMMF_LAUNCH(k_panel_cols, blocks_for(static_cast<i64>(m) * 32, kThreads), kThreads, 0, s, static_cast<i64>(m),
                danch, a.ptr.get(), a.row.get(), a.val.get(), N, Xa.get());
    // pool chunk: panel within a fifth of free memory
    const i64 budget = std::max<i64>(i64{1} << 28, available_bytes() / 5);
    const i64 pc = std::max<i64>(kGemmTJ, std::min<i64>(P, budget / (8 * std::max<i64>(N, 1)) / kGemmTJ * kGemmTJ));
    DBuf<double> Xp(pc * N, s), S(pc * m, s);
    for (i64 p0 = 0; p0 < P; p0 += pc) {
      const i64 n = std::min<i64>(pc, P - p0);
      Xp.zero();
      PMMF_LAUNCH(k_panel_cols, blocks_for(n * 32, kThreads), kThreads, 0, s, n, dpool + p0, a.ptr.get(),
                  a.row.get(), a.val.get(), N, Xp.get());
      dim3 grid(static_cast<unsigned>((n + kGemmTJ - 1) / kGemmTJ), static_cast<unsigned>((m + kGemmTA - 1) / kGemmTA));
      k_score_gemm<<<grid, 256, 0, s>>>(N, static_cast<int>(n), m, Xp.get(), Xa.get(), nb.d_blk.get(), dpn + p0,
                                        dan, rows_mode ? rows_out + p0 * m : S.get());
      launch_counter().fetch_add(1, std::memory_order_relaxed);
      PMMF_CUDA(cudaGetLastError());
      if (!rows_mode)
        PMMF_LAUNCH(k_gemm_argmax, blocks_for(n * 32, kThreads), kThreads, 0, s, n, m, dpool + p0, self.get(),
                    S.get(), assign_out + p0);
    }
    if (trace_enabled()) {
      PMMF_CUDA(cudaStreamSynchronize(s));
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
      std::fprintf(stderr, "[pmmf]   score (gemm): pool=%lld anchors=%d rows=%lld chunk=%lld %.2f ms\n",
                   static_cast<long long>(P), m, static_cast<long long>(N), static_cast<long long>(pc), ms);
    }
    if (!rows_mode) set_self(danch, danch, m, false);
  }
};

__global__ void k_set_self(int m, const int32_t* __restrict__ anchors, const int32_t* __restrict__ pos, bool on,
                           int32_t* __restrict__ self) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a < m) self[anchors[a]] = on ? pos[a] : -1;
}

void Scorer::set_self(const int32_t* anchors, const int32_t* pos, int m, bool on) {
  PMMF_LAUNCH(k_set_self, blocks_for(m, kThreads), kThreads, 0, s, m, anchors, pos, on, self.get());
}

// ------------------------------------------------ device control path
// cluster_recursive (clustering.hpp:85-177) with every O(pool) step on the
// device: the pool's nonzero-norm filter and the final cluster lists are
// stable compactions / a stable radix sort by assignment, unscored columns
// take the round-robin anchor from a scan of the unscored flags, and the
// undersize repair runs as one CTA (below).  The host keeps what the
// reference's RNG stream and recursion order need: the m anchor draws
// (positions only, they do not depend on the values), the m cluster sizes
// and the DFS order of the oversize recursion.

__global__ void k_pool_gather(i64 P, const int32_t* __restrict__ g, const int32_t* __restrict__ g2s,
                              const double* __restrict__ norm_g, int32_t* __restrict__ sid, double* __restrict__ nrm,
                              uint8_t* __restrict__ nz) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= P) return;
  const int32_t x = g[i];
  sid[i] = g2s[x];
  const double v = norm_g[x];
  nrm[i] = v;
  if (nz) nz[i] = v > 0.0 ? 1 : 0;
}

__global__ void k_take(i64 m, const int32_t* __restrict__ src, const int64_t* __restrict__ pos,
                       int32_t* __restrict__ out) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < m) out[i] = src[pos[i]];
}

// Unscored pool columns go round-robin over the anchors in pool order
// (clustering.hpp:124-131): rank among the unscored (exclusive scan) mod m.
__global__ void k_unscored(i64 P, const int32_t* __restrict__ assign, int32_t* __restrict__ flag) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < P) flag[i] = assign[i] < 0 ? 1 : 0;
}
__global__ void k_round_robin(i64 P, int m, const int32_t* __restrict__ rank, int32_t* __restrict__ assign,
                              i64* __restrict__ sizes) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= P) return;
  int32_t a = assign[i];
  if (a < 0) {
    a = rank[i] % m;
    assign[i] = a;
  }
  atomicAdd(reinterpret_cast<unsigned long long*>(sizes + a), 1ull);
}

__global__ void k_cand_flag(i64 P, const int32_t* __restrict__ assign, const i64* __restrict__ sizes, i64 c_min,
                            uint8_t* __restrict__ flag) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < P) flag[i] = sizes[assign[i]] < c_min ? 1 : 0;
}
__global__ void k_cand_take(i64 C, const int64_t* __restrict__ pos, const int32_t* __restrict__ sid,
                            const double* __restrict__ nrm, const int32_t* __restrict__ assign,
                            int32_t* __restrict__ csid, double* __restrict__ cn, int32_t* __restrict__ cur) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= C) return;
  const i64 p = pos[i];
  csid[i] = sid[p];
  cn[i] = nrm[p];
  cur[i] = assign[p];
}
__global__ void k_cand_back(i64 C, const int64_t* __restrict__ pos, const int32_t* __restrict__ cur,
                            int32_t* __restrict__ assign) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < C) assign[pos[i]] = cur[i];
}

// Undersize repair (clustering.hpp:138-163) in one CTA.  Candidates are the
// members of clusters that started below c_min (clusters only grow, so no
// other column can be orphaned), in pool (ascending global) order, with
// their rows of the P_c x m score table.  Per dissolution: the first alive
// cluster of minimal size (ascending index, the reference's alive vector);
// its members = candidates currently in it, in candidate order (= the
// sorted order the reference visits).  An orphan's target does not depend
// on the other orphans' (only the round-robin counter does), so every
// orphan's first strict-max alive anchor with a positive score is found in
// parallel, warp per orphan; thread 0 then assigns them in order, the
// zero-score ones round-robin over the alive list.  State lives in shared
// memory when it fits (sizes, alive list, candidate assignments, orphan
// list, targets), else in the global scratch passed in.
constexpr int kRepairThreads = 1024;
__global__ void __launch_bounds__(kRepairThreads) k_repair(i64 C, int m, i64 c_min, const double* __restrict__ table,
                                                           int32_t* __restrict__ cur_g, i64* __restrict__ sizes_g,
                                                           int32_t* __restrict__ scratch, bool in_smem) {
  using BlockScan = cub::BlockScan<int, kRepairThreads>;
  __shared__ typename BlockScan::TempStorage scan;
  __shared__ int rv[32], ri[32];
  __shared__ int s_worst, s_wpos, s_norph, s_nalive;
  extern __shared__ int32_t rep_smem[];
  int32_t* base = in_smem ? rep_smem : scratch;
  int32_t* sz = base;             // m
  int32_t* alive = sz + m;        // m
  int32_t* cur = alive + m;       // C
  int32_t* orph = cur + C;        // C
  int32_t* res = orph + C;        // C
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  for (int a = tid; a < m; a += blockDim.x) {
    sz[a] = static_cast<int32_t>(sizes_g[a]);
    alive[a] = a;
  }
  for (i64 c = tid; c < C; c += blockDim.x) cur[c] = cur_g[c];
  if (tid == 0) s_nalive = m;
  __syncthreads();
  int orr = 0;  // thread 0's round-robin counter of the current dissolution
  for (;;) {
    const int na = s_nalive;
    if (na <= 1) break;
    // first alive position of minimal size
    int bv = 0x7fffffff, bi = 0x7fffffff;
    for (int i = tid; i < na; i += blockDim.x) {
      const int v = sz[alive[i]];
      if (v < bv || (v == bv && i < bi)) {
        bv = v;
        bi = i;
      }
    }
    for (int o = 16; o; o >>= 1) {
      const int ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov < bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      rv[wid] = bv;
      ri[wid] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < nw; ++w)
        if (rv[w] < bv || (rv[w] == bv && ri[w] < bi)) {
          bv = rv[w];
          bi = ri[w];
        }
      s_wpos = bi;
      s_worst = alive[bi];
    }
    __syncthreads();
    const int worst = s_worst, wpos = s_wpos;
    if (sz[worst] >= c_min) break;
    // erase it from the alive list (order preserved): read, sync, write
    if (na - wpos <= 2 * kRepairThreads) {
      int nxt[2];
      int k = 0;
      for (int i = wpos + tid; i + 1 < na; i += blockDim.x) nxt[k++] = alive[i + 1];
      __syncthreads();
      k = 0;
      for (int i = wpos + tid; i + 1 < na; i += blockDim.x) alive[i] = nxt[k++];
    } else {
      if (tid == 0)
        for (int i = wpos; i + 1 < na; ++i) alive[i] = alive[i + 1];
    }
    // orphans in candidate order: per-thread contiguous chunks + block scan
    const i64 per = (C + blockDim.x - 1) / blockDim.x;
    const i64 c0 = tid * per, c1 = min(C, c0 + per);
    int cnt = 0;
    for (i64 c = c0; c < c1; ++c) cnt += cur[c] == worst;
    int off = 0, total = 0;
    BlockScan(scan).ExclusiveSum(cnt, off, total);
    for (i64 c = c0; c < c1; ++c)
      if (cur[c] == worst) orph[off++] = static_cast<int32_t>(c);
    if (tid == 0) {
      s_norph = total;
      s_nalive = na - 1;
    }
    __syncthreads();
    const int norph = s_norph, nal = na - 1;
    // every orphan's target, warp per orphan
    for (int q = wid; q < norph; q += nw) {
      const double* sr = table + static_cast<i64>(orph[q]) * m;
      double bs = 0.0;
      int bp = 0x7fffffff;
      for (int i = lane; i < nal; i += 32) {
        const double sc = sr[alive[i]];
        if (sc > bs) {  // lanes visit increasing i: strict > keeps the first
          bs = sc;
          bp = i;
        }
      }
      for (int o = 16; o; o >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, bs, o);
        const int op = __shfl_xor_sync(0xffffffffu, bp, o);
        if (os > bs || (os == bs && op < bp)) {
          bs = os;
          bp = op;
        }
      }
      if (lane == 0) res[q] = bs > 0.0 ? bp : -1;
    }
    __syncthreads();
    if (tid == 0) {
      orr = 0;
      for (int q = 0; q < norph; ++q) {
        const int a = res[q] >= 0 ? alive[res[q]] : alive[(orr++) % nal];
        cur[orph[q]] = a;
        ++sz[a];
      }
      sz[worst] = 0;
    }
    __syncthreads();
  }
  for (int a = tid; a < m; a += blockDim.x) sizes_g[a] = sz[a];
  for (i64 c = tid; c < C; c += blockDim.x) cur_g[c] = cur[c];
}

template <typename In, typename T>
void stable_select(In in, const uint8_t* flags, i64 n, T* out, i64* count, cudaStream_t s) {
  DBuf<i64> nsel(1, s);
  size_t tmp = 0;
  PMMF_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, in, flags, out, nsel.get(), static_cast<int64_t>(n), s));
  DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
  PMMF_CUDA(cub::DeviceSelect::Flagged(t.get(), tmp, in, flags, out, nsel.get(), static_cast<int64_t>(n), s));
  *count = nsel.to_host(1)[0];
}

struct DevCtx {
  Scorer* sc;            // one-GPU path
  const SlabSet* ss;     // sharded path (sc == nullptr)
  const Numbering* nb;
  int gemm = -1;         // sharded: the scorer path chosen for the whole matrix
  const int32_t* g2s;    // device: global -> stage id
  const double* norm_g;  // device: norm by global id
  i64 c_min, c_max;
  int d_max;
  int max_depth = 0;
  cudaStream_t s;
};

__global__ void k_own_flags(i64 P, const int32_t* __restrict__ sid, i64 c0, i64 c1, uint8_t* __restrict__ f) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < P) f[i] = sid[i] >= c0 && sid[i] < c1 ? 1 : 0;
}
__global__ void k_take_pos(i64 n, const int64_t* __restrict__ pos, const int32_t* __restrict__ sid,
                           const double* __restrict__ nrm, int32_t* __restrict__ osid, double* __restrict__ on) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  osid[i] = sid[pos[i]];
  on[i] = nrm[pos[i]];
}
__global__ void k_put_assign(i64 n, const int64_t* __restrict__ pos, const int32_t* __restrict__ v,
                             int32_t* __restrict__ out) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < n) out[pos[i]] = v[i];
}
__global__ void k_put_rows(i64 n, int m, const int64_t* __restrict__ pos, const double* __restrict__ v,
                           double* __restrict__ out) {
  const i64 x = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (x >= n * m) return;
  out[pos[x / m] * m + x % m] = v[x];
}

// Scores of a pool against anchors (Scorer::run's contract).  Sharded: the
// anchor columns are gathered to every rank; each rank scores the pool
// columns it owns on its slab plus those anchor columns, with exactly the
// one-GPU kernels, and the results meet by a max over ranks (sentinel -2^31
// for unscored positions, 0.0 in rows mode; scores are >= 0).
void score(DevCtx& ctx, const int32_t* dpool, const double* dpn, i64 P, const int32_t* danch, const double* dan,
           int m, bool rows_mode, int32_t* assign_out, double* rows_out) {
  if (!ctx.ss) {
    ctx.sc->run(dpool, dpn, P, danch, dan, m, rows_mode, assign_out, rows_out);
    return;
  }
  cudaStream_t s = ctx.s;
  const SlabSet& ss = *ctx.ss;
  const Comm& comm = *ss.comm;
  const i64 N = ctx.nb->size();
  Csc anch;
  gather_columns(anch, ss.slabs, ss.own, danch, m, N, comm, s);
  if (rows_mode)
    PMMF_CUDA(cudaMemsetAsync(rows_out, 0, sizeof(double) * P * m, s));
  else
    PMMF_CUDA(cudaMemsetAsync(assign_out, 0x80, sizeof(int32_t) * P, s));
  static const bool st_timing = std::getenv("PMMF_B200_SHARD_TIMING") != nullptr || trace_enabled();
  double tsum = 0.0, tmax = 0.0;
  for (size_t i = 0; i < ss.slabs.size(); ++i) {
    if (st_timing) PMMF_CUDA(cudaStreamSynchronize(s));
    const auto tr0 = std::chrono::steady_clock::now();
    struct Lap {  // per-rank time of this scoring call (scripts/shard_model.py)
      bool on;
      cudaStream_t s;
      std::chrono::steady_clock::time_point t0;
      double *sum, *mx;
      int rank;
      i64* cols;
      ~Lap() {
        if (!on) return;
        cudaStreamSynchronize(s);
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        *sum += ms;
        *mx = std::max(*mx, ms);
        if (std::getenv("PMMF_B200_SHARD_DETAIL"))
          std::fprintf(stderr, "[pmmf]   shard score rank %d: %lld columns %.3f ms\n", rank, static_cast<long long>(*cols),
                       ms);
      }
    };
    i64 Pi = 0;
    Lap lap{st_timing, s, tr0, &tsum, &tmax, ss.comm->local_ranks()[i], &Pi};
    DBuf<uint8_t> f(P, s);
    PMMF_LAUNCH(k_own_flags, blocks_for(P, kThreads), kThreads, 0, s, P, dpool, ss.own[i].first, ss.own[i].second,
                f.get());
    DBuf<int64_t> pos(P, s);
    stable_select(cub::CountingInputIterator<int64_t>(0), f.get(), P, pos.get(), &Pi, s);
    if (Pi == 0) continue;
    DBuf<int32_t> sub(Pi, s);
    DBuf<double> subn(Pi, s);
    PMMF_LAUNCH(k_take_pos, blocks_for(Pi, kThreads), kThreads, 0, s, Pi, pos.get(), dpool, dpn, sub.get(),
                subn.get());
    Csc M;
    merge_columns(M, *ss.slabs[i], anch, s);
    Scorer sc(M, *ctx.nb, s);
    sc.force_gemm = ctx.gemm;
    if (rows_mode) {
      DBuf<double> r(Pi * m, s);
      sc.run(sub.get(), subn.get(), Pi, danch, dan, m, true, nullptr, r.get());
      PMMF_LAUNCH(k_put_rows, blocks_for(Pi * m, kThreads), kThreads, 0, s, Pi, m, pos.get(), r.get(), rows_out);
    } else {
      DBuf<int32_t> as(Pi, s);
      sc.run(sub.get(), subn.get(), Pi, danch, dan, m, false, as.get(), nullptr);
      PMMF_LAUNCH(k_put_assign, blocks_for(Pi, kThreads), kThreads, 0, s, Pi, pos.get(), as.get(), assign_out);
    }
  }
  if (st_timing && comm.virt)
    std::fprintf(stderr, "[pmmf] shard score: %d ranks, sum %.3f ms, max %.3f ms\n", comm.world(), tsum, tmax);
  if (rows_mode)
    allreduce_max_f64(rows_out, P * m, comm, s);
  else
    allreduce_max_i32(assign_out, P, comm, s);
}

// seg: the pool (global ids ascending, device) of one recursion node; on
// return it holds the node's clusters in DFS order and `sizes` has one entry
// per emitted cluster.
void recurse(DevCtx& ctx, int32_t* seg, i64 P, i64 m_request, int depth, Xoshiro& rng, std::vector<i64>& sizes_out) {
  ctx.max_depth = std::max(ctx.max_depth, depth);
  if (P == 0) return;
  cudaStream_t s = ctx.s;
  const auto t_rec = std::chrono::steady_clock::now();
  DBuf<int32_t> sid(P, s), fil(P, s);
  DBuf<double> nrm(P, s);
  DBuf<uint8_t> nz(P, s);
  PMMF_LAUNCH(k_pool_gather, blocks_for(P, kThreads), kThreads, 0, s, P, seg, ctx.g2s, ctx.norm_g, sid.get(), nrm.get(),
              nz.get());
  i64 F = 0;
  stable_select(seg, nz.get(), P, fil.get(), &F, s);
  if (F == 0) {
    sizes_out.push_back(P);
    return;
  }
  // anchors: the partial Fisher-Yates of the reference over the filtered pool
  // (clustering.hpp:99-104) only needs positions
  const i64 m = std::min(m_request, F);
  std::vector<int64_t> slot(static_cast<size_t>(m));
  {
    std::unordered_map<i64, i64> moved;
    auto at = [&](i64 x) {
      auto it = moved.find(x);
      return it == moved.end() ? x : it->second;
    };
    for (i64 t = 0; t < m; ++t) {
      const i64 j = t + static_cast<i64>(rng.uniform_below(static_cast<uint64_t>(F - t)));
      const i64 vt = at(t), vj = at(j);
      moved[t] = vj;
      moved[j] = vt;
    }
    for (i64 t = 0; t < m; ++t) slot[t] = at(t);
  }
  std::vector<int32_t> anchors(static_cast<size_t>(m));
  {
    DBuf<int64_t> dslot(m, s);
    DBuf<int32_t> dan(m, s);
    dslot.upload(slot);
    PMMF_LAUNCH(k_take, blocks_for(m, kThreads), kThreads, 0, s, m, fil.get(), dslot.get(), dan.get());
    anchors = dan.to_host(m);
    std::sort(anchors.begin(), anchors.end());
  }
  DBuf<int32_t> ag(m, s), asid(m, s);
  DBuf<double> anrm(m, s);
  ag.upload(anchors);
  PMMF_LAUNCH(k_pool_gather, blocks_for(m, kThreads), kThreads, 0, s, m, ag.get(), ctx.g2s, ctx.norm_g, asid.get(),
              anrm.get(), static_cast<uint8_t*>(nullptr));
  DBuf<int32_t> assign(P, s);
  const auto t_host0 = std::chrono::steady_clock::now();
  score(ctx, sid.get(), nrm.get(), P, asid.get(), anrm.get(), static_cast<int>(m), false, assign.get(), nullptr);
  if (trace_enabled() && depth == 0) {
    PMMF_CUDA(cudaStreamSynchronize(s));
    std::fprintf(stderr, "[pmmf]     pool setup %.2f ms, scorer %.2f ms\n",
                 std::chrono::duration<double, std::milli>(t_host0 - t_rec).count(),
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_host0).count());
  }
  // round-robin for the unscored, cluster sizes
  DBuf<i64> dsz(m, s);
  dsz.zero();
  {
    DBuf<int32_t> fl(P, s), rk(P, s);
    PMMF_LAUNCH(k_unscored, blocks_for(P, kThreads), kThreads, 0, s, P, assign.get(), fl.get());
    size_t tmp = 0;
    PMMF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, fl.get(), rk.get(), static_cast<int64_t>(P), s));
    DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
    PMMF_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, fl.get(), rk.get(), static_cast<int64_t>(P), s));
    PMMF_LAUNCH(k_round_robin, blocks_for(P, kThreads), kThreads, 0, s, P, static_cast<int>(m), rk.get(), assign.get(),
                dsz.get());
  }
  std::vector<i64> sz = dsz.to_host(m);
  // undersize repair (clustering.hpp:138-163), on the device
  const auto t_repair = std::chrono::steady_clock::now();
  i64 nalive = m;
  if (m > 1 && *std::min_element(sz.begin(), sz.end()) < ctx.c_min) {
    DBuf<uint8_t> cf(P, s);
    PMMF_LAUNCH(k_cand_flag, blocks_for(P, kThreads), kThreads, 0, s, P, assign.get(), dsz.get(), ctx.c_min, cf.get());
    DBuf<int64_t> cpos(P, s);
    i64 C = 0;
    stable_select(cub::CountingInputIterator<int64_t>(0), cf.get(), P, cpos.get(), &C, s);
    DBuf<int32_t> csid(C, s), cur(C, s);
    DBuf<double> cn(C, s), table(C * m, s);
    const size_t rep_bytes = sizeof(int32_t) * static_cast<size_t>(2 * m + 3 * C);
    const bool rep_smem = rep_bytes <= 160 * 1024;
    DBuf<int32_t> rep_scratch(rep_smem ? 1 : 2 * m + 3 * C, s);
    if (rep_smem && rep_bytes > 48 * 1024)
      PMMF_CUDA(cudaFuncSetAttribute(k_repair, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(rep_bytes)));
    PMMF_LAUNCH(k_cand_take, blocks_for(C, kThreads), kThreads, 0, s, C, cpos.get(), sid.get(), nrm.get(),
                assign.get(), csid.get(), cn.get(), cur.get());
    score(ctx, csid.get(), cn.get(), C, asid.get(), anrm.get(), static_cast<int>(m), true, nullptr, table.get());
    PMMF_LAUNCH(k_repair, 1, kRepairThreads, rep_smem ? rep_bytes : 0, s, C, static_cast<int>(m), ctx.c_min,
                table.get(), cur.get(), dsz.get(), rep_scratch.get(), rep_smem);
    PMMF_LAUNCH(k_cand_back, blocks_for(C, kThreads), kThreads, 0, s, C, cpos.get(), cur.get(), assign.get());
    sz = dsz.to_host(m);
    nalive = 0;
    for (i64 a = 0; a < m; ++a) nalive += sz[a] > 0;
  }
  if (trace_enabled() && depth == 0)
    std::fprintf(stderr, "[pmmf]     undersize repair: %lld of %lld clusters alive, %.2f ms\n",
                 static_cast<long long>(nalive), static_cast<long long>(m),
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_repair).count());
  // clusters: a stable sort of the pool by assignment keeps each cluster's
  // members ascending (the reference sorts its grown clusters)
  {
    DBuf<int32_t> k2(P, s), v2(P, s);
    cub::DoubleBuffer<int32_t> kb(assign.get(), k2.get()), vb(seg, v2.get());
    const int bits = std::max(1, bits_for(m));
    size_t tmp = 0;
    PMMF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, static_cast<int64_t>(P), 0, bits, s));
    DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
    PMMF_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, kb, vb, static_cast<int64_t>(P), 0, bits, s));
    if (vb.Current() != seg)
      PMMF_CUDA(cudaMemcpyAsync(seg, vb.Current(), sizeof(int32_t) * P, cudaMemcpyDeviceToDevice, s));
  }
  // oversize recursion (clustering.hpp:165-176) in the alive clusters' order
  i64 off = 0;
  for (i64 a = 0; a < m; ++a) {
    const i64 c = sz[a];
    if (c == 0) continue;
    if (c > ctx.c_max && depth < ctx.d_max)
      recurse(ctx, seg + off, c, (c + ctx.c_max - 1) / ctx.c_max, depth + 1, rng, sizes_out);
    else
      sizes_out.push_back(c);
    off += c;
  }
}

__global__ void k_scatter_norm(i64 P, const int32_t* __restrict__ g, const double* __restrict__ v,
                               double* __restrict__ norm_g, uint8_t* __restrict__ in_pool, bool bypass) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= P) return;
  norm_g[g[i]] = v[i];
  in_pool[i] = (!bypass || v[i] > 0.0) ? 1 : 0;
}
__global__ void k_not(i64 n, const uint8_t* __restrict__ a, uint8_t* __restrict__ b) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < n) b[i] = !a[i];
}
__global__ void k_sid_of(i64 P, const int32_t* __restrict__ g, const int32_t* __restrict__ g2s,
                         int32_t* __restrict__ sid) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < P) sid[i] = g2s[g[i]];
}

}  // namespace

ClusterOut cluster_columns_dev(const SlabSet& ss, const Numbering& nb, const std::vector<i64>& active, i64 n,
                               i64 m_target, i64 c_min, i64 c_max, int d_max, bool bypass, uint64_t seed,
                               cudaStream_t s) {
  if (active.empty()) fail(PMMF_INVALID_ARGUMENT, "cluster_columns: empty active set");
  ClusterOut res;
  // Norms of the active columns (clustering.hpp:189-195), each by its owner.
  const i64 P = static_cast<i64>(active.size());
  DBuf<int32_t> act(P, s), ids(P, s);
  {
    std::vector<int32_t> a32(active.begin(), active.end());
    act.upload(a32);
  }
  PMMF_LAUNCH(k_sid_of, blocks_for(P, kThreads), kThreads, 0, s, P, act.get(), nb.d_g2s.get(), ids.get());
  DBuf<double> dnorm(P, s), norm_g(std::max<i64>(n, 1), s);
  if (ss.sharded()) dnorm.zero();
  for (size_t i = 0; i < ss.slabs.size(); ++i) {
    const Csc& a = *ss.slabs[i];
    const i64 c0 = ss.own[i].first, c1 = ss.own[i].second;
    // columns longer than kLong entries: k_norms_long, a CTA per column
    i64 kLong = 4096;
    if (const char* e = std::getenv("PMMF_B200_NORM_LONG")) kLong = std::atoll(e);  // test hook
    const i64 nblk = nb.clusters();
    const i64 long_len = nblk > 1 ? kLong : (i64{1} << 62);
    PMMF_LAUNCH(k_norms, blocks_for(P * 32, kThreads), kThreads, 0, s, P, ids.get(), a.ptr.get(), a.row.get(),
                a.val.get(), nb.d_blk.get(), dnorm.get(), long_len, c0, c1);
    if (nblk > 1) {
      DBuf<uint8_t> fl(P, s);
      PMMF_LAUNCH(k_long_flags, blocks_for(P, kThreads), kThreads, 0, s, P, ids.get(), a.ptr.get(), long_len, fl.get());
      DBuf<int32_t> lst(P, s);
      i64 nl = 0;
      stable_select(cub::CountingInputIterator<int32_t>(0), fl.get(), P, lst.get(), &nl, s);
      if (nl > 0) {
        DBuf<int64_t> doff(nblk + 1, s);
        doff.upload(nb.off);
        DBuf<double> part(nl * nblk, s);
        PMMF_LAUNCH(k_norms_long, static_cast<unsigned>(nl), kNormLongThreads, 0, s, lst.get(), ids.get(), a.ptr.get(),
                    a.row.get(), a.val.get(), doff.get(), nblk, part.get(), dnorm.get());
      }
    }
  }
  if (ss.sharded()) allreduce_max_f64(dnorm.get(), P, *ss.comm, s);
  norm_g.zero();
  DBuf<uint8_t> in_pool(P, s), byp(P, s);
  PMMF_LAUNCH(k_scatter_norm, blocks_for(P, kThreads), kThreads, 0, s, P, act.get(), dnorm.get(), norm_g.get(),
              in_pool.get(), bypass);
  res.members.alloc(P, s);
  i64 np = 0, nbyp = 0;
  stable_select(act.get(), in_pool.get(), P, res.members.get(), &np, s);
  if (np < P) {  // zero-norm columns bypass (clustering.hpp:207-214), appended by the caller
    PMMF_LAUNCH(k_not, blocks_for(P, kThreads), kThreads, 0, s, P, in_pool.get(), byp.get());
    DBuf<int32_t> bl(P - np, s);
    stable_select(act.get(), byp.get(), P, bl.get(), &nbyp, s);
    std::vector<int32_t> h = bl.to_host(nbyp);
    res.bypassed.assign(h.begin(), h.end());
    PMMF_CUDA(cudaMemcpyAsync(res.members.get() + np, bl.get(), sizeof(int32_t) * nbyp, cudaMemcpyDeviceToDevice, s));
  }
  const auto t_norms = std::chrono::steady_clock::now();
  if (np > 0) {
    std::unique_ptr<Scorer> sc;
    DevCtx ctx{nullptr, nullptr, &nb, -1, nb.d_g2s.get(), norm_g.get(), c_min, c_max, d_max, 0, s};
    if (ss.sharded()) {
      ctx.ss = &ss;
      // the scorer path of the whole matrix (GEMM for dense problems)
      DBuf<int64_t> tot(1, s);
      int64_t mine = 0;
      for (const Csc* a : ss.slabs) mine += a->nnz;
      tot.upload(&mine, 1);
      allreduce_sum_i64(tot.get(), 1, *ss.comm, s);
      const double nnz = static_cast<double>(tot.to_host(1)[0]), N = static_cast<double>(nb.size());
      ctx.gemm = nb.size() > 0 && nnz >= 0.25 * N * N ? 1 : 0;
    } else {
      sc = std::make_unique<Scorer>(*ss.slabs[0], nb, s);
      ctx.sc = sc.get();
    }
    Xoshiro rng(seed);
    recurse(ctx, res.members.get(), np, m_target, 0, rng, res.sizes);
    res.max_depth = ctx.max_depth;
  }
  PMMF_CUDA(cudaStreamSynchronize(s));
  if (trace_enabled())
    std::fprintf(stderr, "[pmmf]   clustering: %.2f ms after norms (pool %lld, nnz %lld)\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_norms).count(),
                 static_cast<long long>(P), static_cast<long long>(ss.slabs[0]->nnz));
  return res;
}

}  // namespace pmmf_b200
