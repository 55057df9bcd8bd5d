// apply.cu — the stage apply A <- Q A Q^T (factorizer.hpp:336-394) as
// column rotation streams, plus the memory-lean transposes between passes.
//
// A pass applies one stage's rotations to the columns of a matrix
// (sparse.hpp:123-156): rotation t on ids (j_0..j_k-1) replaces them by
//   out_a = ((0 + q(a,0) v_0) + q(a,1) v_1) + ...
// over the union support (absent = 0.0), exact zeros dropped (value-neutral,
// SURVEY.md App. A P12).  The row side is the same pass on the transpose
// (App. A P12, "transpose trick").
//
// Scheduling.  Rotations are grouped in dependency levels (search.cu); a
// level's rotations touch disjoint ids.  Every rotation of a level is cut
// into row-range partitions of <= merge_chunk() rows of its longest input, so a
// hub column with 10^6 entries is spread over hundreds of warps instead of
// one.  Each partition is merged twice by one warp: a count pass (kept
// outputs per column), an exclusive scan that yields exact arena offsets,
// then a write pass.  Columns are processed in batches of clusters; a batch
// works in its own arena (superseded versions are garbage), and its final
// columns are copied into a compact Piece, optionally dropping rows that no
// later consumer reads (lean mode).
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <climits>

#include "engine.cuh"

namespace pmmf_b200 {

namespace {

constexpr int kThreads = 256;
// rows of the longest input per partition (PMMF_B200_MERGE_CHUNK, default
// 512; measured on config 4, write + count pass per step: 4096 -> 544 ms,
// 1024 -> 285 ms, 512 -> 257 ms, 256 -> 267 ms)
inline int merge_chunk() {
  const char* e = std::getenv("PMMF_B200_MERGE_CHUNK");
  const int v = e ? std::atoi(e) : 512;
  return v >= 32 ? v : 512;
}

__device__ __forceinline__ int warp_lower_bound(int w, int r) {
  int lo = 0;
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1) {
    const int probe = __shfl_sync(0xffffffffu, w, lo + step - 1);
    if (probe < r) lo += step;
  }
  const int last = __shfl_sync(0xffffffffu, w, lo);
  if (last < r) ++lo;
  return lo;  // number of window rows < r, in [0, 32]
}

__device__ __forceinline__ i64 lower_bound_g(const int32_t* __restrict__ a, i64 lo, i64 hi, int key) {
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

struct PassArgs {
  const int32_t* rots;   // rotation slots of this level
  const int32_t* ids;    // slot x K stage ids (global stage numbering)
  const double* qs;      // slot x K x K
  i64 col0;              // batch column base (local id = stage id - col0)
  const i64* off;        // batch paged table
  const int32_t* len;
  const int32_t* arow;
  const double* aval;
  const int64_t* ioff;   // per level-rotation: first partition index (exclusive scan of nparts)
  int32_t* item_rot;     // partition -> level-rotation index (k_item_rot)
  int chunk;             // partition size (rows of the longest input)
  i64 nrot;              // rotations in level
  i64 nitems;            // total partitions
  int64_t* cnt;          // K * nitems kept counts, layout [K*ioff_t + a*np_t + p]
  int64_t* pos;          // exclusive scan of cnt (write pass; written by the allocation)
  i64 base;              // arena offset of this level's outputs (write pass)
  int32_t* wrow;
  double* wval;
  unsigned long long* out_entries;  // profiling: outputs allocated
  // k = 2 single-partition rotations allocate their own arena space in the
  // write pass (count merge, atomicAdd, write merge back to back)
  unsigned long long* cursor;
  i64 cap;
  int32_t* ovf;
  int level;
  i64* rbase;
  int32_t* rlen;
  // k = 2 count pass: counted partitions per level-rotation; the warp that
  // counts a rotation's last partition allocates it (rot_alloc_warp), so the
  // level needs no separate allocation launch (nullptr: k_rot_alloc runs)
  int32_t* ndone;
  // k = 2: the partition size of this level, chosen by k_level_setup (a level
  // that would leave most warps without a partition is cut finer); nullptr:
  // `chunk` applies
  int32_t* chunk_d;
  int fine_chunk, fine_items;  // rows per partition of a level below fine_items default-size partitions
};

// Row range of partition p of rotation t: split points are rows of the
// longest input at multiples of the chunk.
template <int K>
__device__ void partition_range(const PassArgs& A, int t, i64 p, i64 np, const int* id, i64 (&lo)[K], i64 (&hi)[K]) {
  int longest = 0;
  int Lmax = -1;
#pragma unroll
  for (int b = 0; b < K; ++b) {
    const int L = A.len[id[b]];
    if (L > Lmax) {
      Lmax = L;
      longest = b;
    }
  }
  const i64 lsrc = A.off[id[longest]];
  const int r_lo = p == 0 ? INT_MIN : A.arow[lsrc + p * A.chunk];
  const int r_hi = p == np - 1 ? INT_MAX : A.arow[lsrc + (p + 1) * A.chunk];
#pragma unroll
  for (int b = 0; b < K; ++b) {
    const i64 s = A.off[id[b]], e = s + A.len[id[b]];
    lo[b] = (p == 0) ? s : lower_bound_g(A.arow, s, e, r_lo);
    hi[b] = (p == np - 1) ? e : lower_bound_g(A.arow, s, e, r_hi);
  }
}

// Windowed k-way union merge of one partition, one warp.  kWrite = false
// counts kept outputs per column; true writes them.
template <int K, bool kWrite>
__device__ void merge_partition(const PassArgs& A, const double (&q)[K][K], i64 (&p)[K], const i64 (&hi)[K],
                                int (&kept)[K], const i64 (&dst)[K]) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    int row[K];
    double val[K];
    int frontier = INT_MAX;
    bool any = false;
#pragma unroll
    for (int b = 0; b < K; ++b) {
      const i64 e = p[b] + lane;
      row[b] = e < hi[b] ? A.arow[e] : INT_MAX;
      val[b] = e < hi[b] ? A.aval[e] : 0.0;
      frontier = min(frontier, __shfl_sync(0xffffffffu, row[b], 31));
      any |= p[b] < hi[b];
    }
    if (!any) break;
    bool valid[K];
    int nvalid[K];
#pragma unroll
    for (int b = 0; b < K; ++b) {
      valid[b] = row[b] != INT_MAX && row[b] <= frontier;
      nvalid[b] = __popc(__ballot_sync(0xffffffffu, valid[b]));
    }
    int lb[K][K];
    bool present[K][K];
#pragma unroll
    for (int b = 0; b < K; ++b)
#pragma unroll
      for (int b2 = 0; b2 < K; ++b2) {
        if (b2 == b) {
          lb[b][b2] = lane;
          present[b][b2] = true;
        } else {
          const int l = warp_lower_bound(row[b2], row[b]);
          lb[b][b2] = l;
          // the shuffle must run on all 32 lanes (no short-circuit)
          const int cand = __shfl_sync(0xffffffffu, row[b2], l & 31);
          present[b][b2] = (cand == row[b]) && (l < 32);
        }
      }
    unsigned F[K];
    bool first[K];
#pragma unroll
    for (int b = 0; b < K; ++b) {
      bool f = valid[b];
#pragma unroll
      for (int b2 = 0; b2 < b; ++b2) f = f && !present[b][b2];
      first[b] = f;
      F[b] = __ballot_sync(0xffffffffu, f);
    }
    int rank[K];
    double out[K][K];
#pragma unroll
    for (int b = 0; b < K; ++b) {
      int rk = 0;
#pragma unroll
      for (int b2 = 0; b2 < K; ++b2) {
        const int l = lb[b][b2];
        rk += __popc(F[b2] & (l >= 32 ? 0xffffffffu : ((1u << l) - 1u)));
      }
      rank[b] = rk;
      double v[K];
#pragma unroll
      for (int b2 = 0; b2 < K; ++b2) {
        const double x = __shfl_sync(0xffffffffu, val[b2], lb[b][b2] & 31);
        v[b2] = (b2 == b) ? val[b] : (present[b][b2] ? x : 0.0);
      }
#pragma unroll
      for (int a = 0; a < K; ++a) {
        double acc = 0.0;
#pragma unroll
        for (int b2 = 0; b2 < K; ++b2) acc = dadd(acc, dmul(q[a][b2], v[b2]));
        out[b][a] = acc;
      }
    }
#pragma unroll
    for (int a = 0; a < K; ++a) {
      unsigned words[K];
#pragma unroll
      for (int wd = 0; wd < K; ++wd) {
        unsigned mine = 0;
#pragma unroll
        for (int b = 0; b < K; ++b)
          if (first[b] && out[b][a] != 0.0 && (rank[b] >> 5) == wd) mine |= 1u << (rank[b] & 31);
        words[wd] = __reduce_or_sync(0xffffffffu, mine);
      }
      int total = 0;
#pragma unroll
      for (int wd = 0; wd < K; ++wd) total += __popc(words[wd]);
      if (kWrite) {
#pragma unroll
        for (int b = 0; b < K; ++b) {
          if (first[b] && out[b][a] != 0.0) {
            int pos = 0;
            const int wd = rank[b] >> 5, bit = rank[b] & 31;
#pragma unroll
            for (int x = 0; x < K; ++x)
              if (x < wd) pos += __popc(words[x]);
            pos += __popc(words[wd] & ((1u << bit) - 1u));
            const i64 d = dst[a] + kept[a] + pos;
            A.wrow[d] = row[b];
            A.wval[d] = out[b][a];
          }
        }
      }
      kept[a] += total;
    }
#pragma unroll
    for (int b = 0; b < K; ++b) p[b] += nvalid[b];
  }
}

// k = 2 specialisation of merge_partition (the configs' k).  Outputs are
// the union rows of the two inputs, an exactly-zero result included: the
// reference drops it (sparse.hpp:150), but an explicit 0.0 and an absent
// entry are read identically everywhere downstream (a term q*0.0 in later
// rotations, 0 in Gram and norm sums, nothing in the masses), so keeping
// it is value-neutral -- and it makes the count
// pass a row-only union count: no value loads, no arithmetic.
__device__ __forceinline__ void merge_count2(const PassArgs& A, i64 (&p)[2], const i64 (&hi)[2], int& kept) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    if (p[0] >= hi[0] && p[1] >= hi[1]) break;
    const i64 ea = p[0] + lane, eb = p[1] + lane;
    const int ra = ea < hi[0] ? A.arow[ea] : INT_MAX;
    const int rb = eb < hi[1] ? A.arow[eb] : INT_MAX;
    const int frontier = min(__shfl_sync(0xffffffffu, ra, 31), __shfl_sync(0xffffffffu, rb, 31));
    const bool oka = ra != INT_MAX && ra <= frontier;
    const bool okb = rb != INT_MAX && rb <= frontier;
    const int la = warp_lower_bound(rb, ra);
    const int ca = __shfl_sync(0xffffffffu, rb, la & 31);
    const bool pa = oka && la < 32 && ca == ra;
    const int na = __popc(__ballot_sync(0xffffffffu, oka));
    const int nb = __popc(__ballot_sync(0xffffffffu, okb));
    kept += na + nb - __popc(__ballot_sync(0xffffffffu, pa));
    p[0] += na;
    p[1] += nb;
  }
}

// Write pass: two warp searches (each element's rank in the other window)
// and one ballot of partner-less B rows give every output's position.
// out_a = (0 + q(a,0) v_0) + q(a,1) v_1 with an absent entry read as 0.0.
__device__ __forceinline__ void merge_write2(const PassArgs& A, const double (&q)[2][2], i64 (&p)[2],
                                             const i64 (&hi)[2], int& kept, const i64 (&dst)[2]) {
  const int lane = threadIdx.x & 31;
  const unsigned below = (1u << lane) - 1u;
  for (;;) {
    if (p[0] >= hi[0] && p[1] >= hi[1]) break;
    const i64 ea = p[0] + lane, eb = p[1] + lane;
    const bool ina = ea < hi[0], inb = eb < hi[1];
    const int ra = ina ? A.arow[ea] : INT_MAX;
    const int rb = inb ? A.arow[eb] : INT_MAX;
    const double va = ina ? A.aval[ea] : 0.0;
    const double vb = inb ? A.aval[eb] : 0.0;
    const int frontier = min(__shfl_sync(0xffffffffu, ra, 31), __shfl_sync(0xffffffffu, rb, 31));
    const bool oka = ra != INT_MAX && ra <= frontier;
    const bool okb = rb != INT_MAX && rb <= frontier;
    const int la = warp_lower_bound(rb, ra);  // B-window rows < ra
    const int lb = warp_lower_bound(ra, rb);  // A-window rows < rb
    const int ca = __shfl_sync(0xffffffffu, rb, la & 31);
    const int cb = __shfl_sync(0xffffffffu, ra, lb & 31);
    const double vp = __shfl_sync(0xffffffffu, vb, la & 31);
    const bool pa = la < 32 && ca == ra;               // A element with a B partner
    const bool bonly = okb && !(lb < 32 && cb == rb);  // B element without an A partner
    const unsigned BO = __ballot_sync(0xffffffffu, bonly);
    if (oka) {
      const double x1 = pa ? vp : 0.0;
      const unsigned mb = la >= 32 ? 0xffffffffu : ((1u << la) - 1u);
      const i64 r = kept + lane + __popc(BO & mb);
      A.wrow[dst[0] + r] = ra;
      A.wval[dst[0] + r] = dadd(dadd(0.0, dmul(q[0][0], va)), dmul(q[0][1], x1));
      A.wrow[dst[1] + r] = ra;
      A.wval[dst[1] + r] = dadd(dadd(0.0, dmul(q[1][0], va)), dmul(q[1][1], x1));
    }
    if (bonly) {
      const i64 r = kept + lb + __popc(BO & below);
      A.wrow[dst[0] + r] = rb;
      A.wval[dst[0] + r] = dadd(dadd(0.0, dmul(q[0][0], 0.0)), dmul(q[0][1], vb));
      A.wrow[dst[1] + r] = rb;
      A.wval[dst[1] + r] = dadd(dadd(0.0, dmul(q[1][0], 0.0)), dmul(q[1][1], vb));
    }
    const int na = __popc(__ballot_sync(0xffffffffu, oka));
    kept += na + __popc(BO);
    p[0] += na;
    p[1] += __popc(__ballot_sync(0xffffffffu, okb));
  }
}

// Dense partitions: when every input holds exactly the same contiguous rows
// r0..r0+L-1 (dense clusters: configs 1 and 3), the union merge is the
// identity on the structure and the rotation is elementwise -- a pure
// stream.  Same arithmetic per entry ((0 + q(a,0) v_0) + q(a,1) v_1) + ...;
// outputs keep exact zeros (value-neutral, as on the k = 2 path).
template <int K>
__device__ __forceinline__ int identical_rows(const PassArgs& A, const i64 (&b)[K], const i64 (&e)[K], int& r0) {
  const i64 L = e[0] - b[0];
  if (L <= 0) return -1;
#pragma unroll
  for (int k = 1; k < K; ++k)
    if (e[k] - b[k] != L) return -1;
  r0 = A.arow[b[0]];
  const int r1 = A.arow[e[0] - 1];
  if (static_cast<i64>(r1) - r0 != L - 1) return -1;
#pragma unroll
  for (int k = 1; k < K; ++k)
    if (A.arow[b[k]] != r0 || A.arow[e[k] - 1] != r1) return -1;
  return static_cast<int>(L);
}
template <int K>
__device__ __forceinline__ void write_dense(const PassArgs& A, const double (&q)[K][K], const i64 (&b)[K], int L,
                                            int r0, const i64 (&dst)[K]) {
  for (int i = threadIdx.x & 31; i < L; i += 32) {
    double v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = A.aval[b[k] + i];
#pragma unroll
    for (int a = 0; a < K; ++a) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) acc = dadd(acc, dmul(q[a][k], v[k]));
      A.wrow[dst[a] + i] = r0 + i;
      A.wval[dst[a] + i] = acc;
    }
  }
}

template <int K>
__global__ void k_nparts(PassArgs A, int64_t* __restrict__ nparts, unsigned long long* __restrict__ in_entries) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= A.nrot) return;
  const int t = A.rots[i];
  int Lmax = 0;
  unsigned long long S = 0;
#pragma unroll
  for (int b = 0; b < K; ++b) {
    const int L = A.len[A.ids[static_cast<i64>(t) * K + b] - A.col0];
    Lmax = max(Lmax, L);
    S += static_cast<unsigned long long>(L);
  }
  nparts[i] = max(1, (Lmax + A.chunk - 1) / A.chunk);
  if (A.ndone) A.ndone[i] = 0;
  if (i == 0 && A.chunk_d) *A.chunk_d = A.chunk;
  atomicAdd(in_entries, S);
}

// item_rot[ioff[i] + p] = i for the np_i partitions of level-rotation i, so a
// merge warp finds its rotation with one load instead of a binary search
// over ioff (17 dependent L2 round trips at 10^5 rotations per level).
__global__ void k_item_rot(i64 nrot, const int64_t* __restrict__ ioff, const int64_t* __restrict__ np,
                           int32_t* __restrict__ item_rot) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= nrot) return;
  const i64 b = ioff[i], n = np[i];
  for (i64 p = 0; p < n; ++p) item_rot[b + p] = static_cast<int32_t>(i);
}

// Small levels: k_nparts, the exclusive scan, k_items and k_item_rot in one
// CTA (one launch instead of five; most of a factorization's ~3.7k levels
// have a few hundred rotations).
constexpr int kSetupThreads = 1024;
constexpr i64 kSetupMax = 8 * kSetupThreads;
constexpr int kFineChunk = 128;   // rows per partition of a level below kFineItems default-size partitions
constexpr int kFineItems = 2048;  // (the merge grid holds 4,736 warps)
template <int K>
__global__ void __launch_bounds__(kSetupThreads) k_level_setup(PassArgs A, int64_t* __restrict__ np,
                                                               int64_t* __restrict__ ioff, int64_t* __restrict__ nitems,
                                                               int32_t* __restrict__ item_rot,
                                                               unsigned long long* __restrict__ in_entries,
                                                               PassArgs P, const i64* __restrict__ rbase,
                                                               const int32_t* __restrict__ rlen, i64* __restrict__ off,
                                                               int32_t* __restrict__ len) {
  using BlockScan = cub::BlockScan<int64_t, kSetupThreads>;
  __shared__ typename BlockScan::TempStorage scan;
  __shared__ int64_t s_run;
  __shared__ int s_nq, s_items;
  __shared__ int64_t q_start[kSetupThreads];
  __shared__ int32_t q_len[kSetupThreads], q_rot[kSetupThreads];
  // Most levels fit one tile of kSetupThreads rotations and the launch is a
  // chain of dependent loads (rotation -> ids -> column length, for the commit
  // and again for this level): the first tile's rotation and id loads of both
  // are issued together, before the commit's stores.
  const i64 nrot = A.nrot;
  const i64 i0 = threadIdx.x;
  const bool do_commit = P.nrot > 0 && *reinterpret_cast<volatile const int32_t*>(P.ovf) == INT_MAX;
  int at = -1, pt = -1;
  if (i0 < nrot) at = A.rots[i0];
  if (do_commit && i0 < P.nrot) pt = P.rots[i0];
  int aid[K];
#pragma unroll
  for (int b = 0; b < K; ++b) aid[b] = at >= 0 ? A.ids[static_cast<i64>(at) * K + b] - static_cast<int>(A.col0) : 0;
  // the previous level's commit (k_commit_level), deferred into this launch:
  // its outputs' (off, len) must be in place before this level reads len
  if (pt >= 0) {
#pragma unroll
    for (int a = 0; a < K; ++a) {
      const int id = P.ids[static_cast<i64>(pt) * K + a] - static_cast<int>(P.col0);
      off[id] = rbase[K * i0 + a];
      len[id] = rlen[K * i0 + a];
    }
  }
  if (do_commit)
    for (i64 i = i0 + blockDim.x; i < P.nrot; i += blockDim.x) {
      const int t = P.rots[i];
#pragma unroll
      for (int a = 0; a < K; ++a) {
        const int id = P.ids[static_cast<i64>(t) * K + a] - static_cast<int>(P.col0);
        off[id] = rbase[K * i + a];
        len[id] = rlen[K * i + a];
      }
    }
  __syncthreads();
  // first tile: this thread's rotation, from the ids loaded above
  int Lmax0 = 0;
  unsigned long long Lsum0 = 0;
  if (at >= 0) {
#pragma unroll
    for (int b = 0; b < K; ++b) {
      const int L = A.len[aid[b]];
      Lmax0 = max(Lmax0, L);
      Lsum0 += static_cast<unsigned long long>(L);
    }
  }
  if (threadIdx.x == 0) {
    s_run = 0;
    s_nq = 0;
    s_items = 0;
  }
  unsigned long long ins = 0;
  __syncthreads();
  // Partition size of the level.  With the default size a level of few, short
  // rotations gives most of the grid's warps nothing and its launch lasts as
  // long as one warp's 16-window merge; below kFineItems partitions the level
  // is cut into kFineChunk-row partitions instead (same results for any size).
  int chunk = A.chunk;
  if (A.chunk_d != nullptr && A.chunk <= A.fine_chunk) {
    if (threadIdx.x == 0) *A.chunk_d = chunk;
  } else if (A.chunk_d != nullptr) {
    int mine = at >= 0 ? max(1, (Lmax0 + A.chunk - 1) / A.chunk) : 0;
    for (i64 i = i0 + kSetupThreads; i < nrot; i += kSetupThreads) {
      const int t = A.rots[i];
      int Lmax = 0;
#pragma unroll
      for (int b = 0; b < K; ++b) Lmax = max(Lmax, A.len[A.ids[static_cast<i64>(t) * K + b] - A.col0]);
      mine += max(1, (Lmax + A.chunk - 1) / A.chunk);
    }
    for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&s_items, mine);
    __syncthreads();
    if (s_items < A.fine_items) chunk = A.fine_chunk;
    if (threadIdx.x == 0) *A.chunk_d = chunk;
  }
  for (i64 base = 0; base < nrot; base += kSetupThreads) {
    const i64 i = base + threadIdx.x;
    int64_t v = 0;
    if (i < nrot) {
      int Lmax = Lmax0;
      if (base == 0) {
        ins += Lsum0;
      } else {
        const int t = A.rots[i];
        Lmax = 0;
#pragma unroll
        for (int b = 0; b < K; ++b) {
          const int L = A.len[A.ids[static_cast<i64>(t) * K + b] - A.col0];
          Lmax = max(Lmax, L);
          ins += static_cast<unsigned long long>(L);
        }
      }
      v = max(1, (Lmax + chunk - 1) / chunk);
      np[i] = v;
      if (A.ndone) A.ndone[i] = 0;
    }
    int64_t ex = 0, tot = 0;
    BlockScan(scan).ExclusiveSum(v, ex, tot);
    const int64_t run = s_run;
    if (i < nrot) {
      ioff[i] = run + ex;
      if (v <= 8) {
        for (int64_t q = 0; q < v; ++q) item_rot[run + ex + q] = static_cast<int32_t>(i);
      } else {  // a hub rotation has ~2,000 partitions: filled by a warp below
        const int e = atomicAdd(&s_nq, 1);
        q_start[e] = run + ex;
        q_len[e] = static_cast<int32_t>(v);
        q_rot[e] = static_cast<int32_t>(i);
      }
    }
    __syncthreads();
    const int nq = s_nq;
    for (int e = threadIdx.x >> 5; e < nq; e += kSetupThreads / 32) {
      const int64_t b = q_start[e];
      const int32_t r = q_rot[e];
      for (int q = threadIdx.x & 31; q < q_len[e]; q += 32) item_rot[b + q] = r;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s_run = run + tot;
      s_nq = 0;
    }
    __syncthreads();
  }
  for (int o = 16; o; o >>= 1) ins += __shfl_xor_sync(0xffffffffu, ins, o);
  if ((threadIdx.x & 31) == 0 && ins) atomicAdd(in_entries, ins);
  if (threadIdx.x == 0) *nitems = s_run;
}

// nitems = ioff[nrot-1] + nparts[nrot-1], on the device (no host sync).
__global__ void k_items(i64 nrot, const int64_t* __restrict__ ioff, const int64_t* __restrict__ np,
                        int64_t* __restrict__ nitems) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *nitems = ioff[nrot - 1] + np[nrot - 1];
}

// One warp, k = 2: exclusive scan of rotation i's partition counts (the union
// size, the same for both output columns), one arena allocation of twice the
// total; a partition writes at rbase[2i + b] + pos[2 io + p].  Counts come
// from L2 (ld.cg: other SMs wrote them in this launch), four chunks of 32 in
// flight (a hub rotation has ~2,000 partitions, and this warp is the tail of
// the count pass).
__device__ __forceinline__ void rot_alloc_warp2(const PassArgs& A, i64 i, i64 io, i64 np) {
  const int lane = threadIdx.x & 31;
  const i64 f = 2 * io;
  int64_t* pos = A.pos;
  i64 run = 0;
  for (i64 p0 = 0; p0 < np; p0 += 128) {
    i64 c[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const i64 p = p0 + 32 * j + lane;
      c[j] = p < np ? __ldcg(A.cnt + f + p) : 0;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const i64 p = p0 + 32 * j + lane;
      i64 incl = c[j];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const i64 v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (p < np) pos[f + p] = run + incl - c[j];
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  const i64 all = 2 * run;
  unsigned long long b = 0;
  if (lane == 0) b = atomicAdd(A.cursor, static_cast<unsigned long long>(all));
  b = __shfl_sync(0xffffffffu, b, 0);
  if (static_cast<i64>(b) + all > A.cap) {
    if (lane == 0) atomicMin(A.ovf, A.level);
    return;
  }
  if (lane == 0) {
    atomicAdd(A.out_entries, static_cast<unsigned long long>(all));
    A.rbase[2 * i] = static_cast<i64>(b);
    A.rbase[2 * i + 1] = static_cast<i64>(b) + run;
    A.rlen[2 * i] = static_cast<int32_t>(run);
    A.rlen[2 * i + 1] = static_cast<int32_t>(run);
  }
}

// Per rotation: exclusive scan of its partitions' kept counts per output
// column, one arena allocation (atomicAdd on the cursor) for all K outputs,
// absolute write offsets per partition.  Overflow marks the level as not
// committed; the host compacts and resumes at that level.
template <int K>
__global__ void k_rot_alloc(PassArgs A, const int64_t* __restrict__ nitems_d, unsigned long long* __restrict__ cursor,
                            i64 cap, int32_t* __restrict__ ovf, int level, int64_t* __restrict__ pos,
                            i64* __restrict__ rbase, int32_t* __restrict__ rlen) {
  const i64 i = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= A.nrot || *reinterpret_cast<volatile int32_t*>(ovf) != INT_MAX) return;
  const i64 nitems = *nitems_d;
  const i64 np = (i + 1 < A.nrot ? A.ioff[i + 1] : nitems) - A.ioff[i];
  if (K == 2 && np == 1) return;  // allocated by its write pass
  i64 tot[K];
#pragma unroll
  for (int a = 0; a < K; ++a) {
    const i64 f = K * A.ioff[i] + a * np;
    i64 run = 0;
    for (i64 p0 = 0; p0 < np; p0 += 32) {
      const i64 p = p0 + lane;
      const i64 c = p < np ? A.cnt[f + p] : 0;
      i64 incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const i64 v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (p < np) pos[f + p] = run + incl - c;  // within-column offset
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    tot[a] = run;
  }
  i64 all = 0;
#pragma unroll
  for (int a = 0; a < K; ++a) all += tot[a];
  unsigned long long b = 0;
  if (lane == 0) b = atomicAdd(cursor, static_cast<unsigned long long>(all));
  b = __shfl_sync(0xffffffffu, b, 0);
  if (static_cast<i64>(b) + all > cap) {
    if (lane == 0) atomicMin(ovf, level);
    return;
  }
  if (lane == 0) atomicAdd(A.out_entries, static_cast<unsigned long long>(all));
  i64 col = static_cast<i64>(b);
#pragma unroll
  for (int a = 0; a < K; ++a) {
    const i64 f = K * A.ioff[i] + a * np;
    for (i64 p = lane; p < np; p += 32) pos[f + p] += col;
    if (lane == 0) {
      rbase[K * i + a] = col;
      rlen[K * i + a] = static_cast<int32_t>(tot[a]);
    }
    col += tot[a];
  }
}

template <int K>
__global__ void k_commit_level(PassArgs A, const i64* __restrict__ rbase, const int32_t* __restrict__ rlen,
                               const int32_t* __restrict__ ovf, i64* __restrict__ off, int32_t* __restrict__ len) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= A.nrot || *reinterpret_cast<volatile const int32_t*>(ovf) != INT_MAX) return;
  const int t = A.rots[i];
#pragma unroll
  for (int a = 0; a < K; ++a) {
    const int id = A.ids[static_cast<i64>(t) * K + a] - static_cast<int>(A.col0);
    off[id] = rbase[K * i + a];
    len[id] = rlen[K * i + a];
  }
}

// Persistent variant: warps stride over the level's partitions; the
// partition count is read from the device.
template <int K, bool kWrite>
__global__ void __launch_bounds__(256, K == 2 ? 6 : 2) k_merge_p(PassArgs A, const int64_t* __restrict__ nitems_d, const int32_t* __restrict__ ovf) {
  if (*reinterpret_cast<volatile const int32_t*>(ovf) != INT_MAX) return;
  const i64 nitems = *nitems_d;
  const i64 nw = (static_cast<i64>(gridDim.x) * blockDim.x) >> 5;
  for (i64 item = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5; item < nitems; item += nw) {
    const i64 ri = A.item_rot[item];
    const i64 p = item - A.ioff[ri];
    const i64 np = (ri + 1 < A.nrot ? A.ioff[ri + 1] : nitems) - A.ioff[ri];
    if (K == 2 && np == 1 && !kWrite) continue;  // counted by its own write pass
    const int t = A.rots[ri];
    int id[K];
    double q[K][K];
#pragma unroll
    for (int b = 0; b < K; ++b) {
      id[b] = A.ids[static_cast<i64>(t) * K + b] - static_cast<int>(A.col0);
#pragma unroll
      for (int a = 0; a < K; ++a) q[b][a] = A.qs[(static_cast<i64>(t) * K + b) * K + a];
    }
    i64 beg[K], end[K];
    partition_range<K>(A, t, p, np, id, beg, end);
    int kept[K];
    i64 dst[K];
#pragma unroll
    for (int a = 0; a < K; ++a) {
      kept[a] = 0;
      dst[a] = (kWrite && !(K == 2 && np == 1)) ? A.pos[K * A.ioff[ri] + a * np + p] : 0;
    }
    int r0 = 0;
    const int dl = identical_rows<K>(A, beg, end, r0);
    if (dl >= 0) {
      if (K == 2 && np == 1) {  // self-allocating single partition (below), dense
        unsigned long long b0 = 0;
        if ((threadIdx.x & 31) == 0) b0 = atomicAdd(A.cursor, static_cast<unsigned long long>(K) * dl);
        b0 = __shfl_sync(0xffffffffu, b0, 0);
        if (static_cast<i64>(b0) + static_cast<i64>(K) * dl > A.cap) {
          if ((threadIdx.x & 31) == 0) atomicMin(A.ovf, A.level);
          continue;
        }
        i64 d2[K];
#pragma unroll
        for (int a = 0; a < K; ++a) d2[a] = static_cast<i64>(b0) + static_cast<i64>(a) * dl;
        write_dense<K>(A, q, beg, dl, r0, d2);
        if ((threadIdx.x & 31) == 0) {
#pragma unroll
          for (int a = 0; a < K; ++a) {
            A.rbase[K * ri + a] = d2[a];
            A.rlen[K * ri + a] = dl;
          }
          atomicAdd(A.out_entries, static_cast<unsigned long long>(K) * dl);
        }
        continue;
      }
      if (kWrite) write_dense<K>(A, q, beg, dl, r0, dst);
#pragma unroll
      for (int a = 0; a < K; ++a) kept[a] = dl;
    } else if constexpr (K == 2) {
      if (np == 1) {
        // Single partition: no separate count pass.  Count the union (rows
        // only, the columns are then hot in L1/L2), allocate 2u arena
        // entries, write.  Overflow marks the level uncommitted exactly like
        // k_rot_alloc does; the commit kernel then skips it.
        i64 cb[2] = {beg[0], beg[1]};
        int u = 0;
        merge_count2(A, cb, end, u);
        unsigned long long b0 = 0;
        if ((threadIdx.x & 31) == 0) b0 = atomicAdd(A.cursor, 2ull * static_cast<unsigned long long>(u));
        b0 = __shfl_sync(0xffffffffu, b0, 0);
        if (static_cast<i64>(b0) + 2 * u > A.cap) {
          if ((threadIdx.x & 31) == 0) atomicMin(A.ovf, A.level);
          continue;
        }
        const i64 d2[2] = {static_cast<i64>(b0), static_cast<i64>(b0) + u};
        int w = 0;
        merge_write2(A, q, beg, end, w, d2);
        if ((threadIdx.x & 31) == 0) {
          A.rbase[2 * ri] = d2[0];
          A.rbase[2 * ri + 1] = d2[1];
          A.rlen[2 * ri] = u;
          A.rlen[2 * ri + 1] = u;
          atomicAdd(A.out_entries, 2ull * static_cast<unsigned long long>(u));
        }
        continue;
      }
      int u = 0;  // union size: the same for both output columns
      if (kWrite)
        merge_write2(A, q, beg, end, u, dst);
      else
        merge_count2(A, beg, end, u);
      kept[0] = kept[1] = u;
    } else {
      merge_partition<K, kWrite>(A, q, beg, end, kept, dst);
    }
    if (!kWrite && (threadIdx.x & 31) == 0) {
#pragma unroll
      for (int a = 0; a < K; ++a) A.cnt[K * A.ioff[ri] + a * np + p] = kept[a];
    }
  }
}

// ---- k = 2 merge kernel with latency hiding ------------------------------
// Same results as k_merge_p<2, kWrite> (every output entry, offset and
// count identical), scheduled to keep loads in flight:
//  * item prologue in batches: lane l of a warp resolves the l-th of the
//    warp's next 32 items (item -> rotation -> ids -> column (off, len) ->
//    output offsets, rotation block) into shared memory, so the chain of
//    ~6 dependent global loads is paid once per 32 items, not per item;
//  * partition bounds by a warp-wide search (32 probes per round: 4 rounds
//    for 10^6 entries instead of 20 dependent binary-search loads);
//  * merge windows read from a per-warp shared-memory ring that cp.async
//    fills three or more windows ahead (below).
struct ItemRec {
  i64 off[2];
  i64 dst[2];
  double q[2][2];
  int32_t ri, p, np, len[2], pad;
};
constexpr int kMerge2Warps = kThreads / 32;
// Resident blocks per SM the kernel is compiled for (64 registers).  Measured
// with the ring, write pass per config-4 step: 2: 115.6, 3: 107.1, 4: 106.9,
// 5 (48 registers): 125.5, 6 (40 registers): 159.1 ms.  A two-level window
// search (8 independent pivot probes + 3, a chain of two shuffles instead of
// six) measured 114.5 against 111.1 ms: rejected.
constexpr int kMerge2Occ = 4;
constexpr int kItemBatch = 16;  // items resolved per prologue (<= 32); 11 KB of records per block

// First index i in [lo, hi) with a[i] >= key (hi if none), warp-wide.
__device__ __forceinline__ i64 warp_search_g(const int32_t* __restrict__ a, i64 lo, i64 hi, int key) {
  const int lane = threadIdx.x & 31;
  while (hi - lo > 32) {
    const i64 step = (hi - lo + 31) >> 5;
    const i64 idx = min(lo + (lane + 1) * step, hi) - 1;
    const int c = __popc(__ballot_sync(0xffffffffu, __ldg(a + idx) < key));
    const i64 nlo = lo + c * step;
    hi = min(hi, nlo + step);
    lo = nlo;
    if (c == 32) return hi;
  }
  const i64 e = lo + lane;
  const bool lt = e < hi && __ldg(a + e) < key;
  return lo + __popc(__ballot_sync(0xffffffffu, lt));
}

// ---- merge loops fed from a per-warp shared-memory ring -----------------
// A loop that loads a window once the previous window's advance is known has
// at most one window per input in flight per warp, and the loads' DRAM
// latency sits inside the window-to-window chain (ncu of that variant: 66% of
// the stall samples were long-scoreboard waits on exactly those loads; an L2
// prefetch of the items' inputs did not help: write pass 120.6 ms either way,
// 106.7 ms with the ring).  Here
// each input streams through a ring of four 32-entry chunks filled by
// cp.async (LDGSTS, no registers): chunk c+4 is requested when the window
// leaves chunk c, three or more iterations before its first use, and a window
// is read from shared memory at any alignment.  One commit group per
// iteration; `cp.async.wait_group 2` at the top of an iteration covers every
// chunk the window can touch (an iteration advances an input by <= 32).
constexpr int kRing = 128;  // entries per input: 4 chunks of 32
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// Requests chunk `c` (entries [32c, 32c+32) of the slice) into its ring slot.
template <bool kVals>
__device__ __forceinline__ void ring_issue(uint32_t rs, uint32_t vs, const int32_t* __restrict__ rp,
                                           const double* __restrict__ vp, int c, int h) {
  const int idx = c * 32 + (threadIdx.x & 31);
  if (idx < h) {
    cp_async4(rs + static_cast<uint32_t>(idx & (kRing - 1)) * 4u, rp + idx);
    if (kVals) cp_async8(vs + static_cast<uint32_t>(idx & (kRing - 1)) * 8u, vp + idx);
  }
}

__device__ __forceinline__ int merge_count2_ring(const int32_t* __restrict__ arow, const i64 b0, const i64 b1,
                                                 const i64 e0, const i64 e1, int32_t (*ring_r)[kRing]) {
  const int lane = threadIdx.x & 31;
  const int32_t* __restrict__ rap = arow + b0;
  const int32_t* __restrict__ rbp = arow + b1;
  const int h0 = static_cast<int>(e0 - b0), h1 = static_cast<int>(e1 - b1);
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(ring_r[0]));
  const uint32_t sb = static_cast<uint32_t>(__cvta_generic_to_shared(ring_r[1]));
  __syncwarp();  // the previous item's window reads are done
  ring_issue<false>(sa, 0, rap, nullptr, 0, h0);
  ring_issue<false>(sa, 0, rap, nullptr, 1, h0);
  ring_issue<false>(sb, 0, rbp, nullptr, 0, h1);
  ring_issue<false>(sb, 0, rbp, nullptr, 1, h1);
  cp_async_commit();
  ring_issue<false>(sa, 0, rap, nullptr, 2, h0);
  ring_issue<false>(sb, 0, rbp, nullptr, 2, h1);
  cp_async_commit();
  ring_issue<false>(sa, 0, rap, nullptr, 3, h0);
  ring_issue<false>(sb, 0, rbp, nullptr, 3, h1);
  cp_async_commit();
  int p0 = 0, p1 = 0, c0 = 0, c1 = 0, kept = 0;
  while (p0 < h0 || p1 < h1) {
    cp_async_wait<2>();
    __syncwarp();
    const int ra = p0 + lane < h0 ? ring_r[0][(p0 + lane) & (kRing - 1)] : INT_MAX;
    const int rb = p1 + lane < h1 ? ring_r[1][(p1 + lane) & (kRing - 1)] : INT_MAX;
    const int frontier = min(__shfl_sync(0xffffffffu, ra, 31), __shfl_sync(0xffffffffu, rb, 31));
    const bool oka = ra != INT_MAX && ra <= frontier;
    const bool okb = rb != INT_MAX && rb <= frontier;
    const int na = __popc(__ballot_sync(0xffffffffu, oka));
    const int nb = __popc(__ballot_sync(0xffffffffu, okb));
    p0 += na;
    p1 += nb;
    __syncwarp();  // every lane has read its window before a slot is refilled
    if ((p0 >> 5) > c0) {
      ring_issue<false>(sa, 0, rap, nullptr, c0 + 4, h0);
      ++c0;
    }
    if ((p1 >> 5) > c1) {
      ring_issue<false>(sb, 0, rbp, nullptr, c1 + 4, h1);
      ++c1;
    }
    cp_async_commit();
    const int la = warp_lower_bound(rb, ra);
    const int ca = __shfl_sync(0xffffffffu, rb, la & 31);
    const bool pa = oka && la < 32 && ca == ra;
    kept += na + nb - __popc(__ballot_sync(0xffffffffu, pa));
  }
  cp_async_wait<0>();
  return kept;
}

__device__ __forceinline__ int merge_write2_ring(const PassArgs& A, const double (&q)[2][2], const i64 b0,
                                                 const i64 b1, const i64 e0, const i64 e1, const i64 d0,
                                                 const i64 d1, int32_t (*ring_r)[kRing], double (*ring_v)[kRing]) {
  const int lane = threadIdx.x & 31;
  const unsigned below = (1u << lane) - 1u;
  const int32_t* __restrict__ rap = A.arow + b0;
  const int32_t* __restrict__ rbp = A.arow + b1;
  const double* __restrict__ vap = A.aval + b0;
  const double* __restrict__ vbp = A.aval + b1;
  int32_t* __restrict__ wr0 = A.wrow + d0;
  int32_t* __restrict__ wr1 = A.wrow + d1;
  double* __restrict__ wv0 = A.wval + d0;
  double* __restrict__ wv1 = A.wval + d1;
  const int h0 = static_cast<int>(e0 - b0), h1 = static_cast<int>(e1 - b1);
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(ring_r[0]));
  const uint32_t sb = static_cast<uint32_t>(__cvta_generic_to_shared(ring_r[1]));
  const uint32_t ta = static_cast<uint32_t>(__cvta_generic_to_shared(ring_v[0]));
  const uint32_t tb = static_cast<uint32_t>(__cvta_generic_to_shared(ring_v[1]));
  __syncwarp();  // the previous item's window reads are done
  ring_issue<true>(sa, ta, rap, vap, 0, h0);
  ring_issue<true>(sa, ta, rap, vap, 1, h0);
  ring_issue<true>(sb, tb, rbp, vbp, 0, h1);
  ring_issue<true>(sb, tb, rbp, vbp, 1, h1);
  cp_async_commit();
  ring_issue<true>(sa, ta, rap, vap, 2, h0);
  ring_issue<true>(sb, tb, rbp, vbp, 2, h1);
  cp_async_commit();
  ring_issue<true>(sa, ta, rap, vap, 3, h0);
  ring_issue<true>(sb, tb, rbp, vbp, 3, h1);
  cp_async_commit();
  int p0 = 0, p1 = 0, c0 = 0, c1 = 0, kept = 0;
  while (p0 < h0 || p1 < h1) {
    cp_async_wait<2>();
    __syncwarp();
    const bool ina = p0 + lane < h0, inb = p1 + lane < h1;
    const int ia = (p0 + lane) & (kRing - 1), ib = (p1 + lane) & (kRing - 1);
    const int ra = ina ? ring_r[0][ia] : INT_MAX;
    const int rb = inb ? ring_r[1][ib] : INT_MAX;
    const double va = ina ? ring_v[0][ia] : 0.0;
    const double vb = inb ? ring_v[1][ib] : 0.0;
    const int frontier = min(__shfl_sync(0xffffffffu, ra, 31), __shfl_sync(0xffffffffu, rb, 31));
    const bool oka = ra != INT_MAX && ra <= frontier;
    const bool okb = rb != INT_MAX && rb <= frontier;
    const int na = __popc(__ballot_sync(0xffffffffu, oka));
    const int nb = __popc(__ballot_sync(0xffffffffu, okb));
    p0 += na;
    p1 += nb;
    __syncwarp();  // every lane has read its window before a slot is refilled
    if ((p0 >> 5) > c0) {
      ring_issue<true>(sa, ta, rap, vap, c0 + 4, h0);
      ++c0;
    }
    if ((p1 >> 5) > c1) {
      ring_issue<true>(sb, tb, rbp, vbp, c1 + 4, h1);
      ++c1;
    }
    cp_async_commit();
    const int la = warp_lower_bound(rb, ra);  // B-window rows < ra
    const int lb = warp_lower_bound(ra, rb);  // A-window rows < rb
    const int ca = __shfl_sync(0xffffffffu, rb, la & 31);
    const int cb = __shfl_sync(0xffffffffu, ra, lb & 31);
    const double vp = __shfl_sync(0xffffffffu, vb, la & 31);
    const bool pa = la < 32 && ca == ra;
    const bool bonly = okb && !(lb < 32 && cb == rb);
    const unsigned BO = __ballot_sync(0xffffffffu, bonly);
    if (oka) {
      const double x1 = pa ? vp : 0.0;
      const unsigned mb = la >= 32 ? 0xffffffffu : ((1u << la) - 1u);
      const int r = kept + lane + __popc(BO & mb);
      wr0[r] = ra;
      wv0[r] = dadd(dadd(0.0, dmul(q[0][0], va)), dmul(q[0][1], x1));
      wr1[r] = ra;
      wv1[r] = dadd(dadd(0.0, dmul(q[1][0], va)), dmul(q[1][1], x1));
    }
    if (bonly) {
      const int r = kept + lb + __popc(BO & below);
      wr0[r] = rb;
      wv0[r] = dadd(dadd(0.0, dmul(q[0][0], 0.0)), dmul(q[0][1], vb));
      wr1[r] = rb;
      wv1[r] = dadd(dadd(0.0, dmul(q[1][0], 0.0)), dmul(q[1][1], vb));
    }
    kept += na + __popc(BO);
  }
  cp_async_wait<0>();
  return kept;
}

template <bool kWrite>
__global__ void __launch_bounds__(kThreads, kMerge2Occ) k_merge2(PassArgs A, const int64_t* __restrict__ nitems_d,
                                                        const int32_t* __restrict__ ovf) {
  __shared__ ItemRec recs[kMerge2Warps][kItemBatch];
  __shared__ int32_t ring_r[kMerge2Warps][2][kRing];
  __shared__ double ring_v[kMerge2Warps][2][kWrite ? kRing : 1];
  if (*reinterpret_cast<volatile const int32_t*>(ovf) != INT_MAX) return;
  const i64 nitems = *nitems_d;
  const int chunk = A.chunk_d ? *A.chunk_d : A.chunk;  // this level's partition size (k_level_setup)
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const i64 nw = (static_cast<i64>(gridDim.x) * blockDim.x) >> 5;
  const i64 w = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  ItemRec* rec = recs[wib];
  unsigned long long produced = 0;  // profiling counter, one atomic per warp
  for (i64 first = w; first < nitems; first += kItemBatch * nw) {
    {
      const i64 item = first + lane * nw;
      if (lane < kItemBatch && item < nitems) {
        ItemRec r;
        const int ri = A.item_rot[item];
        const i64 io = A.ioff[ri];
        const i64 io1 = ri + 1 < A.nrot ? A.ioff[ri + 1] : nitems;
        r.ri = ri;
        r.np = static_cast<int32_t>(io1 - io);
        r.p = static_cast<int32_t>(item - io);
        if (kWrite || r.np > 1) {
          const int t = A.rots[ri];
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const int id = A.ids[2 * static_cast<i64>(t) + b] - static_cast<int>(A.col0);
            r.off[b] = A.off[id];
            r.len[b] = A.len[id];
#pragma unroll
            for (int a = 0; a < 2; ++a) r.q[b][a] = A.qs[(2 * static_cast<i64>(t) + b) * 2 + a];
            // fused allocation (A.ndone): one within-column offset per partition + the column's base
            r.dst[b] = !(kWrite && r.np > 1) ? 0
                       : A.ndone            ? A.pos[2 * io + r.p] + A.rbase[2 * static_cast<i64>(ri) + b]
                                            : A.pos[2 * io + b * r.np + r.p];
          }
          if (!kWrite) r.dst[0] = 2 * io;  // count slots of this rotation
        }
        rec[lane] = r;
      }
    }
    __syncwarp();
    const i64 left = (nitems - first + nw - 1) / nw;
    const int cnt = left < kItemBatch ? static_cast<int>(left) : kItemBatch;
    for (int j = 0; j < cnt; ++j) {
      const ItemRec& r = rec[j];
      const int np = r.np, p = r.p, ri = r.ri;
      if (!kWrite && np == 1) continue;  // counted by its own write pass
      const double q[2][2] = {{r.q[0][0], r.q[0][1]}, {r.q[1][0], r.q[1][1]}};
      i64 beg[2], end[2];
      const i64 s0 = r.off[0], s1 = r.off[1];
      const int L0 = r.len[0], L1 = r.len[1];
      if (np == 1) {
        beg[0] = s0;
        end[0] = s0 + L0;
        beg[1] = s1;
        end[1] = s1 + L1;
      } else {
        // partition_range<2>: split rows are rows of the longest input (the
        // first on a tie) at multiples of the chunk
        const int lg = L1 > L0 ? 1 : 0;
        const i64 ls = lg ? s1 : s0;
        const i64 os = lg ? s0 : s1, oe = os + (lg ? L0 : L1);
        const i64 lo_l = ls + static_cast<i64>(p) * chunk;
        const i64 hi_l = p == np - 1 ? ls + (lg ? L1 : L0) : ls + static_cast<i64>(p + 1) * chunk;
        const i64 lo_o = p == 0 ? os : warp_search_g(A.arow, os, oe, __ldg(A.arow + lo_l));
        const i64 hi_o = p == np - 1 ? oe : warp_search_g(A.arow, os, oe, __ldg(A.arow + hi_l));
        beg[0] = lg ? lo_o : lo_l;
        end[0] = lg ? hi_o : hi_l;
        beg[1] = lg ? lo_l : lo_o;
        end[1] = lg ? hi_l : hi_o;
      }
      int r0 = 0;
      const int dl = identical_rows<2>(A, beg, end, r0);
      int u = 0;
      if (dl >= 0) {
        if (np == 1) {  // self-allocating single partition, dense
          unsigned long long b0 = 0;
          if (lane == 0) b0 = atomicAdd(A.cursor, 2ull * static_cast<unsigned long long>(dl));
          b0 = __shfl_sync(0xffffffffu, b0, 0);
          if (static_cast<i64>(b0) + 2 * static_cast<i64>(dl) > A.cap) {
            if (lane == 0) atomicMin(A.ovf, A.level);
            continue;
          }
          const i64 d2[2] = {static_cast<i64>(b0), static_cast<i64>(b0) + dl};
          write_dense<2>(A, q, beg, dl, r0, d2);
          if (lane == 0) {
            A.rbase[2 * ri] = d2[0];
            A.rbase[2 * ri + 1] = d2[1];
            A.rlen[2 * ri] = dl;
            A.rlen[2 * ri + 1] = dl;
          }
          produced += 2ull * static_cast<unsigned long long>(dl);
          continue;
        }
        if (kWrite) write_dense<2>(A, q, beg, dl, r0, r.dst);
        u = dl;
      } else if (np == 1) {
        // single partition: count the union, allocate 2u, write
        u = merge_count2_ring(A.arow, beg[0], beg[1], end[0], end[1], ring_r[wib]);
        unsigned long long b0 = 0;
        if (lane == 0) b0 = atomicAdd(A.cursor, 2ull * static_cast<unsigned long long>(u));
        b0 = __shfl_sync(0xffffffffu, b0, 0);
        if (static_cast<i64>(b0) + 2 * static_cast<i64>(u) > A.cap) {
          if (lane == 0) atomicMin(A.ovf, A.level);
          continue;
        }
        const i64 d0 = static_cast<i64>(b0), d1 = d0 + u;
        if constexpr (kWrite) merge_write2_ring(A, q, beg[0], beg[1], end[0], end[1], d0, d1, ring_r[wib], ring_v[wib]);
        if (lane == 0) {
          A.rbase[2 * ri] = d0;
          A.rbase[2 * ri + 1] = d1;
          A.rlen[2 * ri] = u;
          A.rlen[2 * ri + 1] = u;
        }
        produced += 2ull * static_cast<unsigned long long>(u);
        continue;
      } else if constexpr (kWrite) {
        u = merge_write2_ring(A, q, beg[0], beg[1], end[0], end[1], r.dst[0], r.dst[1], ring_r[wib], ring_v[wib]);
      } else {
        u = merge_count2_ring(A.arow, beg[0], beg[1], end[0], end[1], ring_r[wib]);
      }
      if constexpr (!kWrite) {
        int fin = 0;
        if (lane == 0) {
          A.cnt[r.dst[0] + p] = u;
          if (!A.ndone) A.cnt[r.dst[0] + np + p] = u;
          if (A.ndone) {
            __threadfence();
            fin = atomicAdd(A.ndone + ri, 1) + 1;
          }
        }
        // the warp that counted the rotation's last partition allocates it
        if (__shfl_sync(0xffffffffu, fin, 0) == np) {
          __threadfence();
          if (*reinterpret_cast<volatile const int32_t*>(A.ovf) == INT_MAX) rot_alloc_warp2(A, ri, r.dst[0] >> 1, np);
        }
      }
    }
    __syncwarp();
  }
  if (lane == 0 && produced) atomicAdd(A.out_entries, produced);
}

// ---- persistent level loop ---------------------------------------------
// All dependency levels of a batch in ONE cooperative kernel (the per-level
// chain nparts -> scan -> item map -> count pass -> allocation -> write pass
// -> commit was ~7 launches per level, ~26 k per factorization on config 4).
// Per level, three phases separated by grid barriers:
//   1. partitions per rotation (np) and a block-level scan;
//   2. global offsets of every rotation's partitions, partition -> rotation
//      map, per-item chain state reset;
//   3. merges, one warp per partition (static stride over the items):
//      * single-partition rotations count, allocate (atomicAdd on the arena
//        cursor), write and commit their columns back to back;
//      * multi-partition rotations count their partition, publish it
//        (decoupled look-back over the rotation's partitions: aggregate, then
//        inclusive prefix), write at base + prefix, and the last partition to
//        finish commits.  Partition 0 reserves the rotation's upper bound
//        (K outputs x sum of input lengths), so no separate count pass or
//        allocation kernel is needed; the unused tail of a reservation is
//        garbage that the next compaction drops.
// A look-back only waits on lower items; items are visited in increasing
// order by every warp and all warps are co-resident (cooperative launch), so
// the lowest unfinished item can always proceed.
// Overflow: an allocation that does not fit marks the level (atomicMin);
// rotations that committed are flagged `done` and skipped when the host
// resumes the level after compacting the arena.
struct LoopArgs {
  const int32_t* order;  // plan order (level-sorted slots)
  const i64* lv_lo;      // per level: [lo, hi) into order
  const i64* lv_hi;
  int L0, L1;            // levels [L0, L1]
  const int32_t* ids;
  const double* qs;
  i64 col0;
  i64* off;
  int32_t* len;
  int32_t* arow;
  double* aval;
  int chunk;
  unsigned long long* cursor;
  i64 cap;
  int32_t* ovf;
  uint8_t* done;         // per order position
  int32_t* np;           // per level-rotation
  int64_t* ioff;         // per level-rotation
  int32_t* item_rot;     // per item
  int64_t* bsum;         // per block (+ total)
  int32_t* status;       // per item: 0 none, 1 aggregate, 2 inclusive, 3 failed
  int32_t* agg;          // per item x K
  int32_t* incl;         // per item x K
  i64* rbase;            // per level-rotation: arena base of a multi-partition rotation
  int32_t* ndone;        // per level-rotation: finished partitions
  unsigned long long* in_entries;   // [0] inputs read, [1] outputs written
  i64 max_rot;
};

__device__ __forceinline__ int ld_volatile(const int32_t* p) { return *reinterpret_cast<const volatile int32_t*>(p); }

template <int K>
__device__ void loop_count(const LoopArgs& A, const PassArgs& P, const double (&q)[K][K], const i64 (&beg)[K],
                           const i64 (&end)[K], int (&kept)[K], bool& dense, int& r0) {
  const int dl = identical_rows<K>(P, beg, end, r0);
  dense = dl >= 0;
  if (dense) {
#pragma unroll
    for (int a = 0; a < K; ++a) kept[a] = dl;
    return;
  }
  if constexpr (K == 2) {
    i64 cb[2] = {beg[0], beg[1]};
    int u = 0;
    merge_count2(P, cb, end, u);
    kept[0] = kept[1] = u;
  } else {
    i64 cb[K];
    i64 dst[K];
#pragma unroll
    for (int a = 0; a < K; ++a) {
      cb[a] = beg[a];
      kept[a] = 0;
      dst[a] = 0;
    }
    merge_partition<K, false>(P, q, cb, end, kept, dst);
  }
}

template <int K>
__device__ void loop_write(const PassArgs& P, const double (&q)[K][K], const i64 (&beg)[K], const i64 (&end)[K],
                           bool dense, int r0, const i64 (&dst)[K]) {
  if (dense) {
    write_dense<K>(P, q, beg, static_cast<int>(end[0] - beg[0]), r0, dst);
    return;
  }
  i64 cb[K];
#pragma unroll
  for (int a = 0; a < K; ++a) cb[a] = beg[a];
  if constexpr (K == 2) {
    int u = 0;
    merge_write2(P, q, cb, end, u, dst);
  } else {
    int kept[K];
#pragma unroll
    for (int a = 0; a < K; ++a) kept[a] = 0;
    merge_partition<K, true>(P, q, cb, end, kept, dst);
  }
}

template <int K>
__global__ void __launch_bounds__(256, K == 2 ? 4 : 1) k_level_loop(LoopArgs A) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ int64_t s_scan[256 / 32 + 1];
  __shared__ int64_t s_base;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const i64 gwarp = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const i64 nwarps = (static_cast<i64>(gridDim.x) * blockDim.x) >> 5;
  PassArgs P{};  // the merge helpers' view of the batch
  P.ids = A.ids;
  P.qs = A.qs;
  P.col0 = A.col0;
  P.off = A.off;
  P.len = A.len;
  P.arow = A.arow;
  P.aval = A.aval;
  P.wrow = A.arow;
  P.wval = A.aval;
  P.chunk = A.chunk;
  for (int L = A.L0; L <= A.L1; ++L) {
    const i64 lo = A.lv_lo[L], nrot = A.lv_hi[L] - lo;
    if (nrot <= 0) continue;
    // ---- phase 1: partitions per rotation, block sums over contiguous ranges
    const i64 per = (nrot + gridDim.x - 1) / gridDim.x;
    const i64 b0 = blockIdx.x * per, b1 = min(nrot, b0 + per);
    int64_t mine = 0;
    unsigned long long ins = 0;
    for (i64 i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
      int npi = 0;
      if (!A.done[lo + i]) {
        const int t = A.order[lo + i];
        int Lmax = 0;
#pragma unroll
        for (int b = 0; b < K; ++b) {
          const int l = A.len[A.ids[static_cast<i64>(t) * K + b] - A.col0];
          Lmax = max(Lmax, l);
          ins += static_cast<unsigned long long>(l);
        }
        npi = max(1, (Lmax + A.chunk - 1) / A.chunk);
      }
      A.np[i] = npi;
      mine += npi;
    }
    for (int o = 16; o; o >>= 1) {
      mine += __shfl_xor_sync(0xffffffffu, mine, o);
      ins += __shfl_xor_sync(0xffffffffu, ins, o);
    }
    if (lane == 0 && ins) atomicAdd(A.in_entries, ins);
    if (lane == 0) s_scan[wib] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t t = 0;
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += s_scan[w];
      A.bsum[blockIdx.x] = t;
    }
    grid.sync();
    // ---- phase 2: offsets, item map, chain-state reset
    if (threadIdx.x == 0) {
      int64_t base = 0, all = 0;
      for (unsigned b = 0; b < gridDim.x; ++b) {
        const int64_t v = A.bsum[b];
        if (b < blockIdx.x) base += v;
        all += v;
      }
      s_base = base;
      if (blockIdx.x == 0) A.bsum[gridDim.x] = all;
    }
    __syncthreads();
    {
      // sequential exclusive scan of this block's range, tile by tile
      int64_t run = s_base;
      for (i64 t0 = b0; t0 < b1; t0 += blockDim.x) {
        const i64 i = t0 + threadIdx.x;
        const int v = i < b1 ? A.np[i] : 0;
        // block-wide exclusive scan of v
        int64_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        __syncthreads();
        if (lane == 31) s_scan[wib] = x;
        __syncthreads();
        int64_t wpre = 0, tile = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
          if (w < wib) wpre += s_scan[w];
          tile += s_scan[w];
        }
        if (i < b1) {
          const int64_t o = run + wpre + x - v;
          A.ioff[i] = o;
          for (int p = 0; p < v; ++p) {
            A.item_rot[o + p] = static_cast<int32_t>(i);
            A.status[o + p] = 0;
          }
          A.ndone[i] = 0;
        }
        run += tile;
      }
    }
    grid.sync();
    // ---- phase 3: merges
    const i64 nitems = A.bsum[gridDim.x];
    for (i64 item = gwarp; item < nitems; item += nwarps) {
      const i64 ri = A.item_rot[item];
      const i64 i0 = A.ioff[ri];
      const i64 p = item - i0;
      const int np = A.np[ri];
      const int t = A.order[lo + ri];
      int id[K];
      double q[K][K];
#pragma unroll
      for (int b = 0; b < K; ++b) {
        id[b] = A.ids[static_cast<i64>(t) * K + b] - static_cast<int>(A.col0);
#pragma unroll
        for (int a = 0; a < K; ++a) q[b][a] = A.qs[(static_cast<i64>(t) * K + b) * K + a];
      }
      i64 beg[K], end[K];
      partition_range<K>(P, t, p, np, id, beg, end);
      int kept[K];
      bool dense = false;
      int r0 = 0;
      loop_count<K>(A, P, q, beg, end, kept, dense, r0);
      if (np == 1) {
        int tot = 0;
#pragma unroll
        for (int a = 0; a < K; ++a) tot += kept[a];
        unsigned long long bb = 0;
        if (lane == 0) bb = atomicAdd(A.cursor, static_cast<unsigned long long>(tot));
        bb = __shfl_sync(0xffffffffu, bb, 0);
        if (static_cast<i64>(bb) + tot > A.cap) {
          if (lane == 0) atomicMin(A.ovf, L);
          continue;
        }
        i64 dst[K];
        i64 c = static_cast<i64>(bb);
#pragma unroll
        for (int a = 0; a < K; ++a) {
          dst[a] = c;
          c += kept[a];
        }
        loop_write<K>(P, q, beg, end, dense, r0, dst);
        __syncwarp();
        if (lane == 0) {
#pragma unroll
          for (int a = 0; a < K; ++a) {
            A.off[id[a]] = dst[a];
            A.len[id[a]] = kept[a];
          }
          A.done[lo + ri] = 1;
          atomicAdd(A.in_entries + 1, static_cast<unsigned long long>(tot));
        }
        continue;
      }
      // multi-partition: decoupled look-back over the rotation's partitions
      i64 ub = 0;  // per-output upper bound: sum of the full input lengths
#pragma unroll
      for (int b = 0; b < K; ++b) ub += A.len[id[b]];
      int prefix[K];
#pragma unroll
      for (int a = 0; a < K; ++a) prefix[a] = 0;
      bool failed = false;
      if (lane == 0) {
        if (p == 0) {
          const unsigned long long bb = atomicAdd(A.cursor, static_cast<unsigned long long>(K * ub));
          if (static_cast<i64>(bb) + K * ub > A.cap) {
            atomicMin(A.ovf, L);
            failed = true;
            __threadfence();
            atomicExch(A.status + item, 3);
          } else {
            A.rbase[ri] = static_cast<i64>(bb);
#pragma unroll
            for (int a = 0; a < K; ++a) A.incl[item * K + a] = kept[a];
            __threadfence();
            atomicExch(A.status + item, 2);
          }
        } else {
#pragma unroll
          for (int a = 0; a < K; ++a) A.agg[item * K + a] = kept[a];
          __threadfence();
          atomicExch(A.status + item, 1);
          i64 j = item - 1;
          for (;;) {
            int st = ld_volatile(A.status + j);
            while (st == 0) {
              __nanosleep(64);
              st = ld_volatile(A.status + j);
            }
            __threadfence();
            if (st == 3) {
              failed = true;
              break;
            }
            const int32_t* src = st == 2 ? A.incl : A.agg;
#pragma unroll
            for (int a = 0; a < K; ++a) prefix[a] += ld_volatile(src + j * K + a);
            if (st == 2) break;
            --j;
          }
          if (failed) {
            atomicExch(A.status + item, 3);
          } else {
#pragma unroll
            for (int a = 0; a < K; ++a) A.incl[item * K + a] = prefix[a] + kept[a];
            __threadfence();
            atomicExch(A.status + item, 2);
          }
        }
      }
      failed = __shfl_sync(0xffffffffu, failed, 0);
      if (failed) continue;
#pragma unroll
      for (int a = 0; a < K; ++a) prefix[a] = __shfl_sync(0xffffffffu, prefix[a], 0);
      __threadfence();
      const i64 base = *reinterpret_cast<volatile const i64*>(A.rbase + ri);
      i64 dst[K];
#pragma unroll
      for (int a = 0; a < K; ++a) dst[a] = base + a * ub + prefix[a];
      loop_write<K>(P, q, beg, end, dense, r0, dst);
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        const int fin = atomicAdd(A.ndone + ri, 1);
        if (fin == np - 1) {  // every partition written: commit the rotation
          __threadfence();
          const i64 last = i0 + np - 1;
          int total = 0;
#pragma unroll
          for (int a = 0; a < K; ++a) {
            const int la = ld_volatile(A.incl + last * K + a);
            A.off[id[a]] = base + a * ub;
            A.len[id[a]] = la;
            total += la;
          }
          A.done[lo + ri] = 1;
          atomicAdd(A.in_entries + 1, static_cast<unsigned long long>(total));
        }
      }
    }
    grid.sync();
    if (ld_volatile(A.ovf) != INT_MAX) return;  // the host compacts and resumes
  }
}

__global__ void k_len64(i64 N, const int32_t* __restrict__ len, i64* __restrict__ out) {
  const i64 j = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (j < N) out[j] = len[j];
  if (j == N) out[j] = 0;
}

// Count / copy the live columns of a batch, optionally keeping only rows
// flagged in keep_row (lean mode: rows the next stage reads) unless the
// column itself is flagged in keep_all_col.
// Column segments of <= kSeg entries: per-column kernels over the batch
// arena (final copy, mass count/gather) run warp per segment, so a hub
// column of 10^5-10^6 entries is spread over many warps instead of being
// the tail of the launch.
constexpr int kSeg = 2048;
__global__ void k_seg_n(i64 N, const int32_t* __restrict__ len, i64* __restrict__ nseg) {
  const i64 w = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (w > N) return;
  nseg[w] = w == N ? 0 : max(1, (len[w] + kSeg - 1) / kSeg);
}
__global__ void k_seg_fill(i64 N, const i64* __restrict__ sfirst, int32_t* __restrict__ seg_col) {
  const i64 w = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (w >= N) return;
  for (i64 q = sfirst[w]; q < sfirst[w + 1]; ++q) seg_col[q] = static_cast<int32_t>(w);
}
struct Segs {
  i64 n = 0;
  DBuf<i64> first;      // N + 1: first segment of column w
  DBuf<int32_t> col;    // segment -> column
};
// Entry range of segment q inside its column.
__device__ __forceinline__ void seg_range(const Segs* /*unused*/, i64 q, const int32_t* __restrict__ seg_col,
                                          const i64* __restrict__ sfirst, const int32_t* __restrict__ len, i64& w,
                                          int& b, int& e) {
  w = seg_col[q];
  b = static_cast<int>((q - sfirst[w]) * kSeg);
  e = min(len[w], b + kSeg);
}

__global__ void k_final_count(i64 S, i64 col0, const int32_t* __restrict__ seg_col, const i64* __restrict__ sfirst,
                              const i64* __restrict__ off, const int32_t* __restrict__ len,
                              const int32_t* __restrict__ arow, const uint8_t* __restrict__ keep_row,
                              const uint8_t* __restrict__ keep_all_col, i64* __restrict__ cnt) {
  const i64 q = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q > S) return;
  if (q == S) {
    if (lane == 0) cnt[S] = 0;
    return;
  }
  i64 w;
  int b, e;
  seg_range(nullptr, q, seg_col, sfirst, len, w, b, e);
  const bool all = keep_row == nullptr || (keep_all_col != nullptr && keep_all_col[col0 + w]);
  if (all) {
    if (lane == 0) cnt[q] = e - b;
    return;
  }
  int c = 0;
#pragma unroll 4
  for (int i = b + lane; i < e; i += 32) c += keep_row[arow[off[w] + i]];
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) cnt[q] = c;
}
__global__ void k_final_copy(i64 S, i64 col0, const int32_t* __restrict__ seg_col, const i64* __restrict__ sfirst,
                             const i64* __restrict__ off, const int32_t* __restrict__ len,
                             const int32_t* __restrict__ arow, const double* __restrict__ aval,
                             const uint8_t* __restrict__ keep_row, const uint8_t* __restrict__ keep_all_col,
                             const i64* __restrict__ pos, int32_t* __restrict__ orow, double* __restrict__ oval) {
  const i64 q = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q >= S) return;
  i64 w;
  int b, e;
  seg_range(nullptr, q, seg_col, sfirst, len, w, b, e);
  const bool all = keep_row == nullptr || (keep_all_col != nullptr && keep_all_col[col0 + w]);
  i64 o = pos[q];
  const i64 s = off[w];
  for (int base = b; base < e; base += 128) {  // four windows per round, loads of all four in flight
    int r[4];
    bool k[4];
    double v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = base + 32 * j + lane;
      r[j] = i < e ? arow[s + i] : -1;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      k[j] = r[j] >= 0 && (all || keep_row[r[j]]);
      // dropped rows (most of a row pass's entries): value never read
      v[j] = k[j] ? aval[s + base + 32 * j + lane] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const unsigned m = __ballot_sync(0xffffffffu, k[j]);
      if (k[j]) {
        const i64 d = o + __popc(m & ((1u << lane) - 1u));
        orow[d] = r[j];
        oval[d] = v[j];
      }
      o += __popc(m);
    }
  }
}
// Column pointers of a piece from its segment offsets.
__global__ void k_seg_ptr(i64 N, const i64* __restrict__ sfirst, const i64* __restrict__ spos, i64* __restrict__ ptr) {
  const i64 w = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (w <= N) ptr[w] = spos[sfirst[w]];
}

__global__ void k_paged_init_local(i64 N, const i64* __restrict__ ptr, i64 col0, i64 e0, i64* __restrict__ off,
                                   int32_t* __restrict__ len) {
  const i64 j = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (j >= N) return;
  off[j] = ptr[col0 + j] - e0;
  len[j] = static_cast<int32_t>(ptr[col0 + j + 1] - ptr[col0 + j]);
}

__global__ void k_compact(i64 N, i64* __restrict__ off, const int32_t* __restrict__ len, const i64* __restrict__ pos,
                          const int32_t* __restrict__ r0, const double* __restrict__ v0, int32_t* __restrict__ r1,
                          double* __restrict__ v1) {
  const i64 w = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= N) return;
  const i64 s = off[w], d = pos[w];
  for (int i = lane; i < len[w]; i += 32) {
    r1[d + i] = r0[s + i];
    v1[d + i] = v0[s + i];
  }
  __syncwarp();
  if (lane == 0) off[w] = d;
}

template <typename T>
void exscan(const T* in, T* out, i64 n, cudaStream_t s) {
  size_t tmp = 0;
  PMMF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, static_cast<int64_t>(n), s));
  DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
  PMMF_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, in, out, static_cast<int64_t>(n), s));
}

i64 read_i64(const i64* p, cudaStream_t s) {
  SlowCall slow_("read_i64");
  i64 v = 0;
  PMMF_CUDA(cudaMemcpyAsync(&v, p, sizeof(v), cudaMemcpyDeviceToHost, s));
  PMMF_CUDA(cudaStreamSynchronize(s));
  return v;
}

// Batch working set: paged view of columns [col0, col0+N) in an arena.
struct Batch {
  i64 col0 = 0, N = 0;
  DBuf<i64> off;
  DBuf<int32_t> len;
  DBuf<int32_t> row;
  DBuf<double> val;
  i64 cap = 0, used = 0;

  // Copies the live column versions into a fresh arena of at least
  // `min_cap` entries and 1.5x the live size (peak: old + new arena).
  void compact(i64 min_cap, cudaStream_t s) {
    DBuf<i64> l64(N + 1, s), pos(N + 1, s);
    PMMF_LAUNCH(k_len64, blocks_for(N + 1, kThreads), kThreads, 0, s, N, len.get(), l64.get());
    exscan(l64.get(), pos.get(), N + 1, s);
    const i64 live = read_i64(pos.get() + N, s);
    const i64 ncap = std::max<i64>(min_cap, live + live / 2) + 1024;
    DBuf<int32_t> r1(ncap, s);
    DBuf<double> v1(ncap, s);
    PMMF_LAUNCH(k_compact, blocks_for(N * 32, kThreads), kThreads, 0, s, N, off.get(), len.get(), pos.get(), row.get(),
                val.get(), r1.get(), v1.get());
    row = std::move(r1);
    val = std::move(v1);
    cap = ncap;
    used = live;
  }
};

// ---- residual masses from a batch's final columns (see MassSpec)
// Per column c: the entries of retired rows g that it contributes to the
// mass of g (c taken when it survives or retires after g); the diagonal
// entry (g == c) goes to diag.
// Kept entries (k_final_count) and taken mass entries per segment in one pass
// over the segment's rows; the diagonal entry (g == c) goes to diag.
__global__ void k_final_mass_count(i64 S, i64 col0, const int32_t* __restrict__ seg_col,
                                   const i64* __restrict__ sfirst, const i64* __restrict__ off,
                                   const int32_t* __restrict__ len, const int32_t* __restrict__ arow,
                                   const double* __restrict__ aval, const uint8_t* __restrict__ keep_row,
                                   const uint8_t* __restrict__ keep_all_col, MassSpec M, i64* __restrict__ kcnt,
                                   i64* __restrict__ mcnt) {
  const i64 q = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q > S) return;
  if (q == S) {
    if (lane == 0) {
      kcnt[S] = 0;
      mcnt[S] = 0;
    }
    return;
  }
  i64 w;
  int b, e;
  seg_range(nullptr, q, seg_col, sfirst, len, w, b, e);
  const bool all = keep_row == nullptr || (keep_all_col != nullptr && keep_all_col[col0 + w]);
  const int32_t c = static_cast<int32_t>(col0 + w);
  const int32_t key = M.col_key[c];
  const i64 s0 = off[w];
  int n = 0, kc = 0;
  for (int base = b; base < e; base += 128) {  // four windows per round: rows, then both table gathers
    int32_t g[4], rg[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = base + 32 * j + lane;
      g[j] = i < e ? arow[s0 + i] : -1;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      rg[j] = g[j] >= 0 ? M.row_rank[g[j]] : -1;
      if (!all && g[j] >= 0) kc += keep_row[g[j]];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (rg[j] < 0) continue;
      if (g[j] == c)
        M.diag[rg[j]] = aval[s0 + base + 32 * j + lane];
      else
        n += key > rg[j];
    }
  }
  for (int o = 16; o; o >>= 1) {
    n += __shfl_xor_sync(0xffffffffu, n, o);
    kc += __shfl_xor_sync(0xffffffffu, kc, o);
  }
  if (lane == 0) {
    mcnt[q] = n;
    kcnt[q] = all ? e - b : kc;
  }
}
// Segments [q0, q1) of the batch: (rank of g, v^2) of the taken entries,
// in column order.
__global__ void k_mass_gather(i64 q0, i64 q1, i64 col0, const int32_t* __restrict__ seg_col,
                              const i64* __restrict__ sfirst, const i64* __restrict__ off,
                              const int32_t* __restrict__ len, const int32_t* __restrict__ arow,
                              const double* __restrict__ aval, MassSpec M, const i64* __restrict__ pos,
                              int32_t* __restrict__ okey, double* __restrict__ osq) {
  const i64 q = q0 + ((blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (q >= q1) return;
  i64 w;
  int b, e;
  seg_range(nullptr, q, seg_col, sfirst, len, w, b, e);
  const int32_t c = static_cast<int32_t>(col0 + w);
  const int32_t key = M.col_key[c];
  const i64 s0 = off[w];
  i64 o = pos[q] - pos[q0];
  // four windows per round: rows, rank gathers and values of all four are in
  // flight together (the chain row -> rank -> value was ~3 round trips per window)
  for (int base = b; base < e; base += 128) {
    int32_t g[4], rg[4];
    bool take[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = base + 32 * j + lane;
      g[j] = i < e ? arow[s0 + i] : -1;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) rg[j] = g[j] >= 0 ? M.row_rank[g[j]] : -1;
    double v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      take[j] = rg[j] >= 0 && g[j] != c && key > rg[j];
      v[j] = take[j] ? aval[s0 + base + 32 * j + lane] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const unsigned m = __ballot_sync(0xffffffffu, take[j]);
      if (take[j]) {
        const i64 d = o + __popc(m & ((1u << lane) - 1u));
        okey[d] = static_cast<int32_t>(rg[j] - M.rank_base);
        osq[d] = dmul(v[j], v[j]);
      }
      o += __popc(m);
    }
  }
}
// The chunk is stably sorted by bucket = rank >> shift (so column order is
// kept inside a bucket); one warp per bucket continues the running sums of
// its (1 << shift) ranks in shared memory.  Inside a 32-entry window, equal
// ranks (one per column) are added in lane = column order, one member per
// round (factorizer.hpp:529-542 sequential order).
// start[b] = first sorted position of bucket b (start[nbuckets] = n): one
// streaming pass instead of two 30-step binary searches per bucket warp.
__global__ void k_bucket_bounds(i64 n, i64 nbuckets, int shift, const int32_t* __restrict__ key,
                                i64* __restrict__ start) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i > n) return;
  const i64 prev = i == 0 ? -1 : static_cast<i64>(key[i - 1]) >> shift;
  const i64 cur = i == n ? nbuckets : static_cast<i64>(key[i]) >> shift;
  for (i64 b = prev + 1; b <= cur; ++b) start[b] = i;
}
__global__ void k_mass_buckets(i64 nbuckets, int shift, const int32_t* __restrict__ key,
                               const double* __restrict__ sq, const i64* __restrict__ start, MassSpec M) {
  extern __shared__ double slots[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const i64 bkt = blockIdx.x * static_cast<i64>(blockDim.x >> 5) + wib;
  if (bkt >= nbuckets) return;
  const int width = 1 << shift;
  double* m = slots + static_cast<i64>(wib) * width;
  const i64 r0 = bkt << shift;
  const i64 b = start[bkt], e = start[bkt + 1];
  if (b == e) return;
  double* mass = M.mass + M.rank_base;
  for (int i = lane; i < width; i += 32) m[i] = r0 + i < M.n_retired ? mass[r0 + i] : 0.0;
  __syncwarp();
  int32_t nr = b + lane < e ? key[b + lane] : 0;  // windows loaded one ahead
  double nv = b + lane < e ? sq[b + lane] : 0.0;
  for (i64 x = b; x < e; x += 32) {
    const i64 i = x + lane;
    const bool on = i < e;
    const int32_t r = on ? nr : -1 - lane;  // distinct dummies
    const double v = on ? nv : 0.0;
    if (i + 32 < e) {
      nr = key[i + 32];
      nv = sq[i + 32];
    }
    const unsigned grp = __match_any_sync(0xffffffffu, r);
    const int rk = __popc(grp & ((1u << lane) - 1u));
    const int rounds = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(__popc(grp)));
    for (int k = 0; k < rounds; ++k) {
      if (on && rk == k) m[r - r0] = dadd(m[r - r0], v);
      __syncwarp();
    }
  }
  for (int i = lane; i < width; i += 32)
    if (r0 + i < M.n_retired) mass[r0 + i] = m[i];
}

// Sort-key bits of the mass buckets (PMMF_B200_MASS_KBITS, tuning): fewer
// bits = wider buckets = fewer equal-rank conflicts per 32-entry window, but
// fewer bucket warps.
inline int mass_key_bits() {
  static const int v = [] {
    const char* e = std::getenv("PMMF_B200_MASS_KBITS");
    const int b = e ? std::atoi(e) : 16;
    return b >= 4 && b <= 16 ? b : 16;
  }();
  return v;
}

// Per-batch device scratch for the asynchronous level pipeline.
struct LevelScratch {
  i64 max_rot = 0, max_items = 0;
  DBuf<int64_t> np, ioff, nitems, cnt, pos;
  DBuf<int32_t> item_rot;
  DBuf<i64> rbase;
  DBuf<int32_t> rlen, ovf, ndone, chunk_d;
  DBuf<unsigned long long> cursor, in_entries;
  DBuf<unsigned char> scan_tmp;
  size_t scan_bytes = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;   // profiled write passes
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> cev;  // profiled count passes
  double rot_bytes = 0.0;
};

// Persistent grid of the merge kernels: exactly the resident capacity
// (blocks per SM at this kernel's register use x SMs).  A larger grid runs
// its surplus blocks as a second, thin wave whose statically strided items
// finish last.
// Test hooks, read per call: PMMF_B200_MERGE2=0 sends k = 2 through the
// generic merge kernel, PMMF_B200_FUSED_ALLOC=0 restores the separate
// allocation launch per level.
inline bool merge2_enabled() {
  const char* e = std::getenv("PMMF_B200_MERGE2");
  return !(e && e[0] == '0');
}
inline int fine_param(const char* name, int dflt, int lo, int hi) {
  const char* e = std::getenv(name);
  const int v = e ? std::atoi(e) : dflt;
  return v >= lo && v <= hi ? v : dflt;
}
// k = 2: levels of few partitions are cut finer (PMMF_B200_FINE_LEVELS=0: one size).
inline bool fine_levels_enabled() {
  const char* e = std::getenv("PMMF_B200_FINE_LEVELS");
  return !(e && e[0] == '0');
}
// k = 2: a rotation's arena allocation runs inside the count pass.
inline bool fused_alloc_enabled() {
  const char* e = std::getenv("PMMF_B200_FUSED_ALLOC");
  return !(e && e[0] == '0');
}
template <typename Kernel>
int resident_blocks(Kernel kernel) {
  int per_sm = 0, dev = 0, sms = 148;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0) != cudaSuccess) per_sm = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) (void)cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  (void)cudaGetLastError();
  return std::max(1, per_sm) * sms;
}
template <int K, bool kWrite>
int persistent_blocks(bool merge2) {
  if constexpr (K == 2) {
    if (merge2) {
      static const int nb2 = resident_blocks(k_merge2<kWrite>);
      return nb2;
    }
  }
  static const int nb = resident_blocks(k_merge_p<K, kWrite>);
  return nb;
}

// Opt-in (PMMF_B200_LEVEL_LOOP=1).  Measured on config 4 (gpurun_out r02b,
// DESIGN.md §9): the loop wins only on the small late stages (launch-bound
// levels, stages 11-15: 16.6 -> 10.8 ms) and loses 2x on the large ones
// (stage 1 row-pass levels 142 -> 333 ms): with a static item stride the
// partitions' look-back chains tie the warps' rounds together, so one heavy
// rotation stalls every later item.
inline bool level_loop_enabled() {
  const char* e = std::getenv("PMMF_B200_LEVEL_LOOP");
  return e && e[0] == '1';
}
// Hybrid: the per-level launch chain for the large levels of a batch, then
// one persistent level-loop launch for its tail of levels with fewer than
// this many rotations each (where the chain's ~7 launches per level cost
// more than the loop's three grid barriers).  0 disables.
inline i64 loop_below() {
  const char* e = std::getenv("PMMF_B200_LOOP_BELOW");
  return e ? std::atoll(e) : 0;
}

// Co-resident grid of the level loop (cooperative launch).
template <int K>
int loop_blocks() {
  static const int nb = [] {
    int per_sm = 0, dev = 0, sms = 148;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_level_loop<K>, kThreads, 0) != cudaSuccess)
      per_sm = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) (void)cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    (void)cudaGetLastError();
    return std::max(1, per_sm) * sms;
  }();
  return nb;
}

struct LoopScratch {
  i64 max_rot = 0, max_items = 0;
  DBuf<i64> lv_lo, lv_hi, rbase;
  DBuf<int32_t> np, item_rot, status, agg, incl, ndone;
  DBuf<int64_t> ioff, bsum;
  DBuf<uint8_t> done;
};

template <int K>
void launch_level_loop(LoopArgs A, cudaStream_t s) {
  void* args[] = {&A};
  PMMF_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_level_loop<K>), dim3(loop_blocks<K>()),
                                        dim3(kThreads), args, 0, s));
  launch_counter().fetch_add(1, std::memory_order_relaxed);
}

// The deferred commit of the last level run (run_level), as its own launch.
template <int K>
void flush_commit(Batch& B, LevelScratch& S, PassArgs& pending, cudaStream_t s) {
  if (pending.nrot <= 0) return;
  PMMF_LAUNCH(k_commit_level<K>, blocks_for(pending.nrot, kThreads), kThreads, 0, s, pending, S.rbase.get(),
              S.rlen.get(), S.ovf.get(), B.off.get(), B.len.get());
  pending.nrot = 0;
}

// One dependency level of a batch, entirely on the device (no host sync).
template <int K>
void run_level(Batch& B, LevelScratch& S, const LevelPlan& plan, const int32_t* rots, i64 nrot, int level,
               cudaStream_t s, PassArgs& pending) {
  PassArgs A{};
  A.rots = rots;
  A.ids = plan.ids.get();
  A.qs = plan.q;
  A.col0 = B.col0;
  A.nrot = nrot;
  A.off = B.off.get();
  A.len = B.len.get();
  A.arow = B.row.get();
  A.aval = B.val.get();
  A.wrow = B.row.get();
  A.wval = B.val.get();
  A.ioff = S.ioff.get();
  A.item_rot = S.item_rot.get();
  A.chunk = merge_chunk();
  A.cnt = S.cnt.get();
  A.pos = S.pos.get();
  A.nitems = S.max_items;  // bound; kernels read the exact count from S.nitems
  A.out_entries = S.in_entries.get() + 1;
  A.cursor = S.cursor.get();
  A.cap = B.cap;
  A.ovf = S.ovf.get();
  A.level = level;
  A.rbase = S.rbase.get();
  A.rlen = S.rlen.get();
  const bool merge2 = K == 2 && merge2_enabled();
  A.ndone = (merge2 && fused_alloc_enabled()) ? S.ndone.get() : nullptr;
  A.chunk_d = (merge2 && fine_levels_enabled()) ? S.chunk_d.get() : nullptr;
  A.fine_chunk = fine_param("PMMF_B200_FINE_CHUNK", kFineChunk, 32, 512);
  A.fine_items = fine_param("PMMF_B200_FINE_ITEMS", kFineItems, 1, 8192);
  if (nrot <= kSetupMax && !std::getenv("PMMF_B200_NO_LEVEL_SETUP")) {
    PMMF_LAUNCH(k_level_setup<K>, 1, kSetupThreads, 0, s, A, S.np.get(), S.ioff.get(), S.nitems.get(),
                S.item_rot.get(), S.in_entries.get(), pending, S.rbase.get(), S.rlen.get(), B.off.get(),
                B.len.get());
    pending.nrot = 0;
  } else {
    flush_commit<K>(B, S, pending, s);
    PMMF_LAUNCH(k_nparts<K>, blocks_for(nrot, kThreads), kThreads, 0, s, A, S.np.get(), S.in_entries.get());
    {
      size_t tmp = S.scan_bytes;
      PMMF_CUDA(cub::DeviceScan::ExclusiveSum(S.scan_tmp.get(), tmp, S.np.get(), S.ioff.get(), static_cast<int64_t>(nrot), s));
    }
    PMMF_LAUNCH(k_items, 1, 32, 0, s, nrot, S.ioff.get(), S.np.get(), S.nitems.get());
    PMMF_LAUNCH(k_item_rot, blocks_for(nrot, kThreads), kThreads, 0, s, nrot, S.ioff.get(), S.np.get(),
                S.item_rot.get());
  }
  cudaEvent_t c0 = nullptr, c1 = nullptr;
  if (prof_enabled()) {
    c0 = EventPool::get().take();
    c1 = EventPool::get().take();
    cudaEventRecord(c0, s);
  }
  if (merge2)
    PMMF_LAUNCH(k_merge2<false>, (persistent_blocks<K, false>(true)), kThreads, 0, s, A, S.nitems.get(), S.ovf.get());
  else
    PMMF_LAUNCH((k_merge_p<K, false>), (persistent_blocks<K, false>(false)), kThreads, 0, s, A, S.nitems.get(),
                S.ovf.get());
  if (c0) {
    cudaEventRecord(c1, s);
    S.cev.push_back({c0, c1});
  }
  if (!A.ndone)  // else allocated inside the count pass (rot_alloc_warp)
    PMMF_LAUNCH(k_rot_alloc<K>, blocks_for(nrot * 32, kThreads), kThreads, 0, s, A, S.nitems.get(), S.cursor.get(), B.cap,
                S.ovf.get(), level, S.pos.get(), S.rbase.get(), S.rlen.get());
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (prof_enabled()) {
    e0 = EventPool::get().take();
    e1 = EventPool::get().take();
    cudaEventRecord(e0, s);
  }
  if (merge2)
    PMMF_LAUNCH(k_merge2<true>, (persistent_blocks<K, true>(true)), kThreads, 0, s, A, S.nitems.get(), S.ovf.get());
  else
    PMMF_LAUNCH((k_merge_p<K, true>), (persistent_blocks<K, true>(false)), kThreads, 0, s, A, S.nitems.get(),
                S.ovf.get());
  if (e0) {
    cudaEventRecord(e1, s);
    S.ev.push_back({e0, e1});
    S.rot_bytes += static_cast<double>(nrot) * (8.0 * K * K + 4.0 * K);
  }
  pending = A;  // committed by the next level's setup (or flush_commit)
}

__global__ void k_gather_ptr(i64 n, const i64* __restrict__ src, const i64* __restrict__ idx, i64* __restrict__ dst) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

__global__ void k_plan(const int32_t* __restrict__ nrot, const int64_t* __restrict__ base,
                       const int64_t* __restrict__ coff, const int32_t* __restrict__ rot_loc,
                       const int32_t* __restrict__ rot_level, int k, int32_t* __restrict__ ids,
                       int32_t* __restrict__ lvl) {
  const int u = blockIdx.x;
  const i64 b = base[u];
  for (int t = threadIdx.x; t < nrot[u]; t += blockDim.x) {
    const i64 sl = b + t;
    for (int a = 0; a < k; ++a) ids[sl * k + a] = static_cast<int32_t>(coff[u] + rot_loc[sl * k + a]);
    lvl[sl] = rot_level[sl];
  }
}
__global__ void k_iota(i64 n, int32_t* __restrict__ x) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < n) x[i] = static_cast<int32_t>(i);
}
__global__ void k_level_bounds(i64 n, const int32_t* __restrict__ lv, int maxl, i64* __restrict__ start) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i > n) return;
  const int prev = i == 0 ? -1 : lv[i - 1];
  const int cur = i == n ? maxl + 1 : lv[i];
  for (int L = prev + 1; L <= cur; ++L) start[L] = i;
}

}  // namespace

// Level plan of a stage (rotation slots sorted by dependency level; stable,
// so slots stay ascending inside a level).
void build_plan(LevelPlan& plan, const SearchOut& so, const DBuf<int64_t>& out_base,
                const DBuf<int64_t>& cluster_off, i64 nclusters, i64 R, int k, cudaStream_t s) {
  plan.R = R;
  plan.k = k;
  plan.q = so.rot_q.get();
  plan.max_level = 0;
  plan.level_start.assign(1, 0);
  plan.h_order.clear();
  if (R == 0 || nclusters == 0) return;
  plan.ids.alloc(R * k, s);
  DBuf<int32_t> lvl(R, s), slot(R, s), lvl2(R, s);
  lvl.zero();
  PMMF_LAUNCH(k_plan, static_cast<unsigned>(nclusters), 256, 0, s, so.nrot.get(), out_base.get(), cluster_off.get(),
              so.rot_loc.get(), so.rot_level.get(), k, plan.ids.get(), lvl.get());
  PMMF_LAUNCH(k_iota, blocks_for(R, kThreads), kThreads, 0, s, R, slot.get());
  plan.order.alloc(R, s);
  {
    size_t tmp = 0;
    PMMF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, lvl.get(), lvl2.get(), slot.get(), plan.order.get(),
                                              static_cast<int64_t>(R), 0, 31, s));
    DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
    PMMF_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, lvl.get(), lvl2.get(), slot.get(), plan.order.get(),
                                              static_cast<int64_t>(R), 0, 31, s));
  }
  int maxl = 0;
  PMMF_CUDA(cudaMemcpyAsync(&maxl, lvl2.get() + R - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  PMMF_CUDA(cudaStreamSynchronize(s));
  plan.max_level = maxl;
  DBuf<i64> start(maxl + 2, s);
  PMMF_LAUNCH(k_level_bounds, blocks_for(R + 1, kThreads), kThreads, 0, s, R, lvl2.get(), maxl, start.get());
  std::vector<i64> h = start.to_host(maxl + 2);
  plan.level_start.assign(h.begin() + 1, h.end());  // level L occupies [level_start[L-1], level_start[L])
  plan.h_order = plan.order.to_host(R);
}

namespace {
// Masses of the retired rows over the final columns of batch B, in column
// chunks of <= chunk_nnz taken entries (ascending column order).
void build_segs(const Batch& B, Segs& G, cudaStream_t s) {
  DBuf<i64> nseg(B.N + 1, s);
  G.first.alloc(B.N + 1, s);
  PMMF_LAUNCH(k_seg_n, blocks_for(B.N + 1, kThreads), kThreads, 0, s, B.N, B.len.get(), nseg.get());
  exscan(nseg.get(), G.first.get(), B.N + 1, s);
  G.n = read_i64(G.first.get() + B.N, s);
  G.col.alloc(std::max<i64>(G.n, 1), s);
  PMMF_LAUNCH(k_seg_fill, blocks_for(B.N, kThreads), kThreads, 0, s, B.N, G.first.get(), G.col.get());
}

void batch_masses(const Batch& B, const Segs& G, const MassSpec& M, const DBuf<i64>& cnt, cudaStream_t s) {
  const bool tr = trace_enabled();
  double tms[4] = {0, 0, 0, 0};
  auto tl = std::chrono::steady_clock::now();
  auto lap = [&](int k) {
    if (!tr) return;
    PMMF_CUDA(cudaStreamSynchronize(s));
    const auto now = std::chrono::steady_clock::now();
    tms[k] += std::chrono::duration<double, std::milli>(now - tl).count();
    tl = now;
  };
  const i64 S = G.n;
  DBuf<i64> pos(S + 1, s);  // cnt: taken entries per segment (k_final_mass_count)
  exscan(cnt.get(), pos.get(), S + 1, s);
  const std::vector<i64> hp = pos.to_host(S + 1);
  if (hp[S] == 0) return;
  const i64 chunk = std::max<i64>(kSeg, std::min<i64>(M.chunk_nnz, i64{1} << 30));
  const i64 cap = std::min<i64>(hp[S], chunk);
  // buckets of 2^shift ranks: a 16-bit sort key (two radix passes)
  const int rb = std::max(1, bits_for(std::max<i64>(M.n_retired - 1, 1)));
  const int shift = std::max(0, rb - mass_key_bits());
  const int kbits = rb - shift;
  const i64 nbuckets = ((M.n_retired - 1) >> shift) + 1;
  DBuf<int32_t> k1, k2;
  DBuf<double> v1, v2;
  DBuf<unsigned char> tmp;
  DBuf<i64> bstart(nbuckets + 1, s);
  i64 have = 0;
  auto ensure = [&](i64 n) {
    if (n <= have) return;
    k1.alloc(n, s);
    k2.alloc(n, s);
    v1.alloc(n, s);
    v2.alloc(n, s);
    size_t a = 0;
    cub::DoubleBuffer<int32_t> kd(k1.get(), k2.get());
    cub::DoubleBuffer<double> vd(v1.get(), v2.get());
    PMMF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, a, kd, vd, static_cast<int64_t>(n), shift, shift + kbits, s));
    tmp.alloc(static_cast<i64>(a) + 1, s);
    have = n;
  };
  ensure(cap);
  lap(0);
  constexpr int kWarpsPerBlock = 8;
  const size_t smem = static_cast<size_t>(kWarpsPerBlock) * (size_t{1} << shift) * sizeof(double);
  int nchunks = 0;
  i64 w0 = 0;  // segments [w0, w1) per chunk (a segment holds <= kSeg <= chunk entries)
  while (w0 < S) {
    i64 w1 = w0 + 1;
    while (w1 < S && hp[w1 + 1] - hp[w0] <= chunk) ++w1;
    const i64 n = hp[w1] - hp[w0];
    if (n > 0) {
      ensure(n);
      ++nchunks;
      PMMF_LAUNCH(k_mass_gather, blocks_for((w1 - w0) * 32, kThreads), kThreads, 0, s, w0, w1, B.col0, G.col.get(),
                  G.first.get(), B.off.get(), B.len.get(), B.row.get(), B.val.get(), M, pos.get(), k1.get(), v1.get());
      lap(1);
      cub::DoubleBuffer<int32_t> kd(k1.get(), k2.get());
      cub::DoubleBuffer<double> vd(v1.get(), v2.get());
      size_t t = static_cast<size_t>(tmp.n);
      PMMF_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), t, kd, vd, static_cast<int64_t>(n), shift, shift + kbits, s));
      lap(2);
      PMMF_LAUNCH(k_bucket_bounds, blocks_for(n + 1, kThreads), kThreads, 0, s, n, nbuckets, shift, kd.Current(),
                  bstart.get());
      PMMF_LAUNCH(k_mass_buckets, blocks_for(nbuckets * 32, 32 * kWarpsPerBlock), 32 * kWarpsPerBlock, smem, s,
                  nbuckets, shift, kd.Current(), vd.Current(), bstart.get(), M);
      lap(3);
    }
    w0 = w1;
  }
  if (tr)
    std::fprintf(stderr, "[pmmf]     masses: %lld taken in %d chunks: count %.1f gather %.1f sort %.1f sums %.1f ms\n",
                 static_cast<long long>(hp[S]), nchunks, tms[0], tms[1], tms[2], tms[3]);
}
}  // namespace

void rotate_pass(std::vector<Piece>& out, const Csc& in, const std::vector<i64>& off,
                 const std::vector<i64>& slot_base, const LevelPlan& plan, const uint8_t* keep_row,
                 const uint8_t* keep_all_col, i64 batch_nnz, double growth, const MassSpec* ms,
                 cudaStream_t s, i64 u_lo, i64 u_hi) {
  out.clear();
  const i64 m = u_hi < 0 ? static_cast<i64>(off.size()) - 1 : u_hi;
  // host copy of ptr at cluster boundaries: one gather kernel and one copy
  // (a copy per cluster was 513 synchronous 8-byte transfers, ~5 ms per pass)
  std::vector<i64> eptr(static_cast<size_t>(m + 1), 0);
  {
    const i64 cnt = m - u_lo + 1;
    DBuf<i64> didx(cnt, s), dval(cnt, s);
    didx.upload(off.data() + u_lo, cnt);
    PMMF_LAUNCH(k_gather_ptr, blocks_for(cnt, kThreads), kThreads, 0, s, cnt, in.ptr.get(), didx.get(), dval.get());
    dval.download(eptr.data() + u_lo, cnt);
    PMMF_CUDA(cudaStreamSynchronize(s));
  }
  i64 u0 = u_lo;
  while (u0 < m) {
    i64 u1 = u0 + 1;
    while (u1 < m && eptr[u1 + 1] - eptr[u0] <= batch_nnz) ++u1;
    Batch B;
    B.col0 = off[u0];
    B.N = off[u1] - off[u0];
    const i64 e0 = eptr[u0], ne = eptr[u1] - eptr[u0];
    B.cap = std::max<i64>(static_cast<i64>(static_cast<double>(ne) * std::max(growth, 2.0)), ne + (i64{1} << 22));
    B.used = ne;
    B.off.alloc(std::max<i64>(B.N, 1), s);
    B.len.alloc(std::max<i64>(B.N, 1), s);
    B.row.alloc(B.cap, s);
    B.val.alloc(B.cap, s);
    if (ne) {
      PMMF_CUDA(cudaMemcpyAsync(B.row.get(), in.row.get() + e0, sizeof(int32_t) * ne, cudaMemcpyDeviceToDevice, s));
      PMMF_CUDA(cudaMemcpyAsync(B.val.get(), in.val.get() + e0, sizeof(double) * ne, cudaMemcpyDeviceToDevice, s));
    }
    PMMF_LAUNCH(k_paged_init_local, blocks_for(B.N, kThreads), kThreads, 0, s, B.N, in.ptr.get(), B.col0, e0,
                B.off.get(), B.len.get());
    // levels restricted to the batch's rotation slots: the plan's order is
    // sorted by (level, slot), so the batch's slots are a contiguous
    // sub-range of every level (found on the host copy)
    const i64 sb = slot_base[u0], se = slot_base[u1];
    std::vector<std::pair<i64, i64>> range(static_cast<size_t>(plan.max_level) + 1, {0, 0});
    i64 max_rot = 1;
    for (int L = 1; L <= plan.max_level && se > sb; ++L) {
      const i64 b = plan.level_start[L - 1], e = plan.level_start[L];
      if (e <= b) continue;
      const i64 lo = std::lower_bound(plan.h_order.begin() + b, plan.h_order.begin() + e, static_cast<int32_t>(sb)) -
                     plan.h_order.begin();
      const i64 hi = std::lower_bound(plan.h_order.begin() + b, plan.h_order.begin() + e, static_cast<int32_t>(se)) -
                     plan.h_order.begin();
      range[L] = {lo, hi};
      max_rot = std::max(max_rot, hi - lo);
    }
    LevelScratch S;
    const int K = plan.k;
    auto size_items = [&] {
      // + the finest cut of a small level (k_level_setup): fewer than
      // fine_items default-size partitions, each at most chunk / fine_chunk + 1 finer ones
      S.max_items = max_rot + B.cap / merge_chunk() + 1 +
                    static_cast<i64>(fine_param("PMMF_B200_FINE_ITEMS", kFineItems, 1, 8192)) *
                        (merge_chunk() / fine_param("PMMF_B200_FINE_CHUNK", kFineChunk, 32, 512) + 1);
      S.cnt.alloc(K * S.max_items, s);
      S.pos.alloc(K * S.max_items, s);
      S.item_rot.alloc(S.max_items, s);
    };
    S.max_rot = max_rot;
    S.np.alloc(max_rot, s);
    S.ioff.alloc(max_rot + 1, s);
    S.nitems.alloc(1, s);
    S.rbase.alloc(K * max_rot, s);
    S.rlen.alloc(K * max_rot, s);
    S.ndone.alloc(max_rot, s);
    S.chunk_d.alloc(1, s);
    S.ovf.alloc(1, s);
    S.cursor.alloc(1, s);
    S.in_entries.alloc(2, s);
    S.in_entries.zero();
    {
      PMMF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, S.scan_bytes, S.np.get(), S.ioff.get(),
                                              static_cast<int64_t>(max_rot), s));
      S.scan_tmp.alloc(static_cast<i64>(S.scan_bytes) + 1, s);
    }
    const bool loop = level_loop_enabled();
    const i64 below = loop ? 0 : loop_below();
    int L_switch = plan.max_level + 1;  // hybrid: levels >= L_switch all below the threshold
    if (below > 0)
      while (L_switch > 1 && range[L_switch - 1].second - range[L_switch - 1].first < below) --L_switch;
    const bool hybrid = below > 0 && L_switch <= plan.max_level;
    if (!loop) size_items();
    auto set_scalar = [&](auto& buf, auto v) {
      PMMF_CUDA(cudaMemcpyAsync(buf.get(), &v, sizeof(v), cudaMemcpyHostToDevice, s));
      PMMF_CUDA(cudaStreamSynchronize(s));
    };
    set_scalar(S.ovf, static_cast<int32_t>(INT_MAX));
    set_scalar(S.cursor, static_cast<unsigned long long>(ne));
    int Lstart = 1, repeat = 0, last_ovf = -1;
    const bool tr = trace_enabled();
    auto tb = std::chrono::steady_clock::now();
    double t_levels = 0.0, t_compact = 0.0;
    auto since = [&](std::chrono::steady_clock::time_point& t0) {
      PMMF_CUDA(cudaStreamSynchronize(s));
      const auto now = std::chrono::steady_clock::now();
      const double ms = std::chrono::duration<double, std::milli>(now - t0).count();
      t0 = now;
      return ms;
    };
    // persistent level loop (default) or the per-level launch chain
    LoopScratch X;
    int loop_grid = 0;
    if (loop || hybrid) {
      switch (K) {
        case 2: loop_grid = loop_blocks<2>(); break;
        case 3: loop_grid = loop_blocks<3>(); break;
        case 4: loop_grid = loop_blocks<4>(); break;
        case 5: loop_grid = loop_blocks<5>(); break;
        case 6: loop_grid = loop_blocks<6>(); break;
        case 7: loop_grid = loop_blocks<7>(); break;
        case 8: loop_grid = loop_blocks<8>(); break;
        default: fail(PMMF_INVALID_ARGUMENT, "apply: unsupported k");
      }
      std::vector<i64> hlo(static_cast<size_t>(plan.max_level) + 1, 0), hhi(hlo.size(), 0);
      for (int L = 1; L <= plan.max_level; ++L) {
        hlo[L] = range[L].first;
        hhi[L] = range[L].second;
        if (L >= (loop ? 1 : L_switch))  // the chain counts its own levels (run_level)
          S.rot_bytes += static_cast<double>(range[L].second - range[L].first) * (8.0 * K * K + 4.0 * K);
      }
      X.lv_lo.alloc(static_cast<i64>(hlo.size()), s);
      X.lv_hi.alloc(static_cast<i64>(hhi.size()), s);
      X.lv_lo.upload(hlo);
      X.lv_hi.upload(hhi);
      X.max_rot = max_rot;
      X.np.alloc(max_rot, s);
      X.ioff.alloc(max_rot, s);
      X.rbase.alloc(max_rot, s);
      X.ndone.alloc(max_rot, s);
      X.bsum.alloc(loop_grid + 1, s);
      X.done.alloc(std::max<i64>(plan.R, 1), s);
      X.done.zero();
    }
    auto size_loop_items = [&] {
      X.max_items = max_rot + B.cap / merge_chunk() + 1;
      X.item_rot.alloc(X.max_items, s);
      X.status.alloc(X.max_items, s);
      X.agg.alloc(K * X.max_items, s);
      X.incl.alloc(K * X.max_items, s);
    };
    if (loop || hybrid) size_loop_items();
    auto launch_loop = [&](int L0) {
        LoopArgs LA{};
        LA.order = plan.order.get();
        LA.lv_lo = X.lv_lo.get();
        LA.lv_hi = X.lv_hi.get();
        LA.L0 = L0;
        LA.L1 = plan.max_level;
        LA.ids = plan.ids.get();
        LA.qs = plan.q;
        LA.col0 = B.col0;
        LA.off = B.off.get();
        LA.len = B.len.get();
        LA.arow = B.row.get();
        LA.aval = B.val.get();
        LA.chunk = merge_chunk();
        LA.cursor = S.cursor.get();
        LA.cap = B.cap;
        LA.ovf = S.ovf.get();
        LA.done = X.done.get();
        LA.np = X.np.get();
        LA.ioff = X.ioff.get();
        LA.item_rot = X.item_rot.get();
        LA.bsum = X.bsum.get();
        LA.status = X.status.get();
        LA.agg = X.agg.get();
        LA.incl = X.incl.get();
        LA.rbase = X.rbase.get();
        LA.ndone = X.ndone.get();
        LA.in_entries = S.in_entries.get();
        LA.max_rot = max_rot;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (prof_enabled()) {
          e0 = EventPool::get().take();
          e1 = EventPool::get().take();
          cudaEventRecord(e0, s);
        }
        switch (K) {
          case 2: launch_level_loop<2>(LA, s); break;
          case 3: launch_level_loop<3>(LA, s); break;
          case 4: launch_level_loop<4>(LA, s); break;
          case 5: launch_level_loop<5>(LA, s); break;
          case 6: launch_level_loop<6>(LA, s); break;
          case 7: launch_level_loop<7>(LA, s); break;
          case 8: launch_level_loop<8>(LA, s); break;
          default: fail(PMMF_INVALID_ARGUMENT, "apply: unsupported k");
        }
        if (e0) {
          cudaEventRecord(e1, s);
          S.ev.push_back({e0, e1});
        }
    };
    for (;;) {
      if (loop) {
        launch_loop(Lstart);
      } else {
        PassArgs pending{};  // the last level's deferred commit
        auto flush = [&] {
          switch (K) {
            case 2: flush_commit<2>(B, S, pending, s); break;
            case 3: flush_commit<3>(B, S, pending, s); break;
            case 4: flush_commit<4>(B, S, pending, s); break;
            case 5: flush_commit<5>(B, S, pending, s); break;
            case 6: flush_commit<6>(B, S, pending, s); break;
            case 7: flush_commit<7>(B, S, pending, s); break;
            case 8: flush_commit<8>(B, S, pending, s); break;
            default: fail(PMMF_INVALID_ARGUMENT, "apply: unsupported k");
          }
        };
        for (int L = Lstart; L <= plan.max_level; ++L) {
          if (hybrid && L >= L_switch) {
            flush();
            launch_loop(L);
            break;
          }
          const auto [lo, hi] = range[L];
          if (hi <= lo) continue;
          const int32_t* rots = plan.order.get() + lo;
          switch (K) {
            case 2: run_level<2>(B, S, plan, rots, hi - lo, L, s, pending); break;
            case 3: run_level<3>(B, S, plan, rots, hi - lo, L, s, pending); break;
            case 4: run_level<4>(B, S, plan, rots, hi - lo, L, s, pending); break;
            case 5: run_level<5>(B, S, plan, rots, hi - lo, L, s, pending); break;
            case 6: run_level<6>(B, S, plan, rots, hi - lo, L, s, pending); break;
            case 7: run_level<7>(B, S, plan, rots, hi - lo, L, s, pending); break;
            case 8: run_level<8>(B, S, plan, rots, hi - lo, L, s, pending); break;
            default: fail(PMMF_INVALID_ARGUMENT, "apply: unsupported k");
          }
        }
        flush();
      }
      int32_t ovf = 0;
      PMMF_CUDA(cudaMemcpyAsync(&ovf, S.ovf.get(), sizeof(ovf), cudaMemcpyDeviceToHost, s));
      PMMF_CUDA(cudaStreamSynchronize(s));
      if (tr) t_levels += since(tb);
      if (ovf == INT_MAX) break;
      // Level `ovf` did not fit: nothing of it was committed.  Compact the
      // live columns into a larger arena and resume there.
      // Same-size arena when most of it was superseded versions; doubled
      // while the same level keeps failing.
      repeat = ovf == last_ovf ? repeat + 1 : 0;
      last_ovf = ovf;
      B.compact(std::max<i64>(B.cap << std::min(repeat, 8), i64{1} << 22), s);
      if (trace_enabled())
        std::fprintf(stderr, "[pmmf]   arena overflow at level %d: compacted to %lld live, cap %lld\n", ovf,
                     static_cast<long long>(B.used), static_cast<long long>(B.cap));
      if (loop || hybrid) size_loop_items();
      if (!loop) size_items();
      set_scalar(S.cursor, static_cast<unsigned long long>(B.used));
      set_scalar(S.ovf, static_cast<int32_t>(INT_MAX));
      Lstart = ovf;
      if (tr) t_compact += since(tb);
    }
    if (prof_enabled() && !S.ev.empty()) {
      double ms = 0.0;
      for (auto& [e0, e1] : S.ev) {
        float t = 0.f;
        cudaEventElapsedTime(&t, e0, e1);
        ms += t;
        EventPool::get().give(e0);
        EventPool::get().give(e1);
      }
      std::vector<unsigned long long> io = S.in_entries.to_host(2);
      // algorithmic bytes: inputs read once, outputs written
      // once (12 B per entry), rotation blocks (8k^2 + 4k per rotation)
      prof_add_n(loop ? "rotate_loop" : "rotate_write", static_cast<int64_t>(S.ev.size()), ms,
                 12.0 * static_cast<double>(io[0] + io[1]) + S.rot_bytes);
      double cms = 0.0;
      for (auto& [e0, e1] : S.cev) {
        float t = 0.f;
        cudaEventElapsedTime(&t, e0, e1);
        cms += t;
        EventPool::get().give(e0);
        EventPool::get().give(e1);
      }
      // count pass bytes: the row indices of the multi-partition inputs (not
      // counted separately; reported as 4 B per input entry, an upper bound)
      prof_add_n("rotate_count", static_cast<int64_t>(S.cev.size()), cms, 4.0 * static_cast<double>(io[0]));
    }
    double t_mass = 0.0;
    Segs G;
    build_segs(B, G, s);
    DBuf<i64> cnt(G.n + 1, s), spos(G.n + 1, s);
    if (ms) {
      // kept-entry and taken-entry counts per segment in one pass over the rows
      DBuf<i64> mcnt(G.n + 1, s);
      PMMF_LAUNCH(k_final_mass_count, blocks_for((G.n + 1) * 32, kThreads), kThreads, 0, s, G.n, B.col0, G.col.get(),
                  G.first.get(), B.off.get(), B.len.get(), B.row.get(), B.val.get(), keep_row, keep_all_col, *ms,
                  cnt.get(), mcnt.get());
      batch_masses(B, G, *ms, mcnt, s);
      if (tr) t_mass = since(tb);
    } else {
      PMMF_LAUNCH(k_final_count, blocks_for((G.n + 1) * 32, kThreads), kThreads, 0, s, G.n, B.col0, G.col.get(),
                  G.first.get(), B.off.get(), B.len.get(), B.row.get(), keep_row, keep_all_col, cnt.get());
    }
    // finalize into a compact piece
    Piece P;
    P.c0 = B.col0;
    P.c1 = B.col0 + B.N;
    P.ptr.alloc(B.N + 1, s);
    exscan(cnt.get(), spos.get(), G.n + 1, s);
    PMMF_LAUNCH(k_seg_ptr, blocks_for(B.N + 1, kThreads), kThreads, 0, s, B.N, G.first.get(), spos.get(), P.ptr.get());
    P.nnz = read_i64(spos.get() + G.n, s);
    P.row.alloc(std::max<i64>(P.nnz, 1), s);
    P.val.alloc(std::max<i64>(P.nnz, 1), s);
    PMMF_LAUNCH(k_final_copy, blocks_for(G.n * 32, kThreads), kThreads, 0, s, G.n, B.col0, G.col.get(), G.first.get(),
                B.off.get(), B.len.get(), B.row.get(), B.val.get(), keep_row, keep_all_col, spos.get(), P.row.get(),
                P.val.get());
    if (tr)
      std::fprintf(stderr, "[pmmf]     batch cols %lld: levels %.1f compact %.1f masses %.1f final %.1f ms (nnz in %lld out %lld)\n",
                   static_cast<long long>(B.N), t_levels, t_compact, t_mass, since(tb), static_cast<long long>(ne),
                   static_cast<long long>(P.nnz));
    out.push_back(std::move(P));
    u0 = u1;
  }
}

}  // namespace pmmf_b200
