// search.cu — randomized greedy k-tuple pivot search (Algorithm 2,
// factorizer.hpp:198-319), one CTA per cluster, all clusters of a stage in
// one launch.
//
// Per cluster the state is the dense column-major Gram tile G_u and diagonal
// block D_u (full storage: the conjugated k x k corner is not bitwise
// symmetric), the active set as a bitmask in shared
// memory, and the diagonals of G and D in shared memory.
//
// The loop is latency-bound (one rotation depends on the previous one), so
// an iteration is organised around three barriers and three dependent global
// round trips:
//   * every thread advances its own copy of the cluster's RNG stream (P5)
//     and every warp selects the idx-th active index from the bitmask, so the
//     draw needs no broadcast;
//   * the CTA scans column `draw` of G (loads issued before use) for the best
//     partner(s) (score g^2 / G_ll, strict >, ties to the lowest index; P8)
//     -> barrier 1;
//   * warp 0 loads the k x k corners of G and D, builds q =
//     rotation_from_gram (P9) in registers, writes the conjugated corners
//     back (P10), picks the victim (P11), retires it and records the rotation
//     with its dependency level for the stage apply -> barrier 2;
//   * the CTA rewrites the k columns (coalesced) and mirrored rows of G and D
//     over every off-corner row -> barrier 3.
// Everything is exact fp64 without contraction (-fmad=false).
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <numeric>

#include "engine.cuh"
#include "rng.cuh"
#include "rotation.cuh"

namespace pmmf_b200 {

namespace {

constexpr int kSearchThreads = 512;
constexpr int kWarps = kSearchThreads / 32;

struct Best {
  double s;
  int l;
};
__device__ __forceinline__ bool better(double s, int l, double bs, int bl) {
  return s > bs || (s == bs && l < bl);
}

// idx-th set bit (0-based) of the bitmask; executed by one full warp.
__device__ int warp_select(const uint32_t* bits, int nwords, int idx) {
  const int lane = threadIdx.x & 31;
  const int per = (nwords + 31) / 32;
  const int w0 = lane * per, w1 = min(nwords, w0 + per);
  int cnt = 0;
  for (int w = w0; w < w1; ++w) cnt += __popc(bits[w]);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int excl = incl - cnt;
  int found = -1;
  if (idx >= excl && idx < incl) {
    int rem = idx - excl;
    for (int w = w0; w < w1; ++w) {
      uint32_t b = bits[w];
      const int pc = __popc(b);
      if (rem < pc) {
        for (int t = 0; t < rem; ++t) b &= b - 1;
        found = w * 32 + (__ffs(b) - 1);
        break;
      }
      rem -= pc;
    }
  }
  const unsigned who = __ballot_sync(0xffffffffu, found >= 0);
  return __shfl_sync(0xffffffffu, found, who ? __ffs(who) - 1 : 0);
}

// Same selection through per-group counts (group = 32 words = 1024 ids, at
// most 32 groups): two warp scans instead of a scan over every word.
__device__ int warp_select2(const uint32_t* bits, const int* gcnt, int nwords, int idx) {
  const int lane = threadIdx.x & 31;
  const int ngroups = (nwords + 31) >> 5;
  const int gc = lane < ngroups ? gcnt[lane] : 0;
  int incl = gc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int g = __ffs(__ballot_sync(0xffffffffu, idx < incl)) - 1;
  const int rem = idx - __shfl_sync(0xffffffffu, incl - gc, g);
  const int w = (g << 5) + lane;
  const uint32_t word = w < nwords ? bits[w] : 0u;
  const int pc = __popc(word);
  int incl2 = pc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl2, o);
    if (lane >= o) incl2 += v;
  }
  const int wl = __ffs(__ballot_sync(0xffffffffu, rem < incl2)) - 1;
  int r2 = rem - __shfl_sync(0xffffffffu, incl2 - pc, wl);
  uint32_t ww = __shfl_sync(0xffffffffu, word, wl);
  for (; r2 > 0; --r2) ww &= ww - 1;
  return ((g << 5) + wl) * 32 + (__ffs(ww) - 1);
}

__device__ __forceinline__ bool is_on(const uint32_t* bits, int l) { return (bits[l >> 5] >> (l & 31)) & 1u; }

struct KArgs {
  const int64_t* c;
  const int64_t* tile;
  const int64_t* budget;
  const uint64_t* seed;
  const int64_t* out_base;
  double eta;
  double* G;
  double* D;
  double* diag_scratch;    // 2 * max_c per cluster when the diagonals do not fit in shared memory
  int32_t* level_scratch;  // max_c per cluster
  i64 max_c;
  bool diag_in_smem;
  int32_t* nrot;
  int32_t* nelim;
  int32_t* rot_loc;
  double* rot_q;
  int32_t* rot_level;
  int32_t* elim_loc;
  int32_t* error;
  unsigned long long* timing;  // optional: 8 clock64 phase totals per cluster
  const int32_t* order;        // CTA -> cluster, largest clusters first (LPT)
};

template <int K>
__global__ void __launch_bounds__(kSearchThreads, 2) k_search(KArgs A) {
  extern __shared__ unsigned char smem[];
  __shared__ Best red[2][kWarps];
  __shared__ int sh_loc[K];
  __shared__ double sh_q[K][K];
  __shared__ int sh_victim;
  __shared__ int sh_oldts[K];
  const int u = A.order[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const i64 c64 = A.c[u];
  if (c64 < K) {
    if (tid == 0) {
      A.nrot[u] = 0;
      A.nelim[u] = 0;
    }
    return;
  }
  const int c = static_cast<int>(c64);
  const i64 base = A.out_base[u];
  i64 budget = static_cast<i64>(floor(A.eta * static_cast<double>(c)));
  if (A.budget[u] >= 0) budget = min(budget, A.budget[u]);
  const int nwords = (c + 31) / 32;
  uint32_t* bits = reinterpret_cast<uint32_t*>(smem);
  double* gd;
  double* dd;
  if (A.diag_in_smem) {
    gd = reinterpret_cast<double*>(smem + ((static_cast<size_t>(nwords) * 4 + 15) / 16) * 16);
  } else {
    gd = A.diag_scratch + static_cast<i64>(u) * 3 * A.max_c;
  }
  dd = gd + c;
  // ts[i]: rotation counter of the last rotation that rewrote column i.
  // Entry (row a, column b) lives in column b, unless a was rotated later
  // than b, in which case it lives in column a (at row b): the reference's
  // mirror write (sparse.hpp:433-439) stores the same value in both places,
  // and corner pairs (equal ts) keep their own, possibly asymmetric, copy.
  // So no strided mirror writes are needed.
  int32_t* ts = reinterpret_cast<int32_t*>(dd + c);
  int32_t* level = A.level_scratch + static_cast<i64>(u) * A.max_c;
  double* G = A.G + A.tile[u];
  double* D = A.D + A.tile[u];
  __shared__ int gcnt[32];
  const bool sel2 = nwords <= 1024;
  for (int w = tid; w < nwords; w += kSearchThreads) {
    const int hi = min(32, c - w * 32);
    bits[w] = hi == 32 ? 0xffffffffu : ((1u << hi) - 1u);
  }
  if (tid < 32) gcnt[tid] = max(0, min(1024, c - tid * 1024));
  for (int l = tid; l < c; l += kSearchThreads) {
    gd[l] = G[static_cast<i64>(l) * c + l];
    dd[l] = D[static_cast<i64>(l) * c + l];
    ts[l] = 0;
    level[l] = 0;
  }
  Xoshiro rng(A.seed[u]);  // every thread advances an identical copy
  int count = c, nrot = 0, nelim = 0, par = 0;
  unsigned long long tacc[6] = {0, 0, 0, 0, 0, 0}, tprev = clock64();
#define TMARK(i)                                   \
  if (A.timing && tid == 0) {                      \
    const unsigned long long now_ = clock64();     \
    tacc[i] += now_ - tprev;                       \
    tprev = now_;                                  \
  }
  __syncthreads();

  for (i64 s = 0; s < budget; ++s) {
    if (count <= K - 1) break;
    const int idx = static_cast<int>(rng.uniform_below(static_cast<uint64_t>(count)));
    const int draw = sel2 ? warp_select2(bits, gcnt, nwords, idx) : warp_select(bits, nwords, idx);
    TMARK(0)
    if (gd[draw] <= 0.0) {  // vanished column: retire without a rotation (:234-238)
      __syncthreads();      // everyone has read bits for this draw
      if (tid == 0) {
        bits[draw >> 5] &= ~(1u << (draw & 31));
        gcnt[(draw >> 10) & 31] -= 1;
        A.elim_loc[base + nelim] = draw;
      }
      --count;
      ++nelim;
      __syncthreads();
      continue;
    }
    // ---- partners (:243-280)
    int loc[K];
    loc[0] = draw;
    int npart = 0;
    const double* gcol = G + static_cast<i64>(draw) * c;
    const int tsd = ts[draw];
#pragma unroll 1
    for (int round = 0; round < K - 1; ++round) {
      double bs = 0.0;
      int bl = INT_MAX;
      for (int l0 = tid; l0 < c; l0 += 4 * kSearchThreads) {
        double gv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          // G(l, draw): column draw, or column l when l was rotated later
          const int l = l0 + j * kSearchThreads;
          gv[j] = 0.0;
          if (l < c && is_on(bits, l))
            gv[j] = ts[l] > tsd ? G[static_cast<i64>(l) * c + draw] : gcol[l];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int l = l0 + j * kSearchThreads;
          if (l >= c || l == draw || !is_on(bits, l)) continue;
          const double nl = gd[l];
          if (nl <= 0.0) continue;
          bool taken = false;
#pragma unroll
          for (int t = 1; t < K; ++t) taken |= (t <= round) && loc[t] == l;
          if (taken) continue;
          const double sc = (gv[j] * gv[j]) / nl;
          if (sc > 0.0 && better(sc, l, bs, bl)) {
            bs = sc;
            bl = l;
          }
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, bs, o);
        const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
        if (better(os, ol, bs, bl)) {
          bs = os;
          bl = ol;
        }
      }
      if (lane == 0) red[par][wid] = Best{bs, bl};
      __syncthreads();
      Best b = red[par][0];
#pragma unroll
      for (int w = 1; w < kWarps; ++w)
        if (better(red[par][w].s, red[par][w].l, b.s, b.l)) b = red[par][w];
      par ^= 1;
      if (!(b.s > 0.0)) break;
#pragma unroll
      for (int t = 1; t < K; ++t)
        if (t == round + 1) loc[t] = b.l;
      ++npart;
    }
    if (npart < K - 1) {
      // Fill with the lowest active indices not yet chosen (:256, :275-279);
      // every warp computes the same answer.
      int have = npart;
      for (int i = 0; have < K - 1; ++i) {
        const int l = sel2 ? warp_select2(bits, gcnt, nwords, i) : warp_select(bits, nwords, i);
        bool taken = l == draw;
#pragma unroll
        for (int t = 1; t < K; ++t) taken |= (t <= have) && loc[t] == l;
        if (!taken) {
#pragma unroll
          for (int t = 1; t < K; ++t)
            if (t == have + 1) loc[t] = l;
          ++have;
        }
      }
    }
    TMARK(1)
    // ---- rotation + corners + victim (warp 0; lane 0 writes)
    if (wid == 0) {
      double gs[K][K], cd[K][K], q[K][K], ng[K][K], nd[K][K];
#pragma unroll
      for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = 0; b < K; ++b) {
          // entry (row loc[a], column loc[b]) under the timestamp rule
          const bool rowcol = ts[loc[a]] > ts[loc[b]];
          const i64 at = rowcol ? static_cast<i64>(loc[a]) * c + loc[b] : static_cast<i64>(loc[b]) * c + loc[a];
          gs[a][b] = G[at];
          cd[a][b] = D[at];
        }
      const bool ok = rotation_from_gram_k<K>(gs, q);
      conjugate_corner_k<K>(q, gs, ng);
      conjugate_corner_k<K>(q, cd, nd);
      int victim = -1;
      double vn = 0.0;
#pragma unroll
      for (int a = 1; a < K; ++a) {
        const double off = off_diag_norm_sq(ng[a][a], nd[a][a]);
        if (victim < 0 || off < vn) {
          victim = loc[a];
          vn = off;
        }
      }
      if (off_diag_norm_sq(ng[0][0], nd[0][0]) < vn) victim = draw;
      __syncwarp();  // every lane has read the corner before lane 0 rewrites it
      if (lane == 0) {
        if (!ok) atomicExch(A.error, 1);
#pragma unroll
        for (int a = 0; a < K; ++a) {
          sh_loc[a] = loc[a];
#pragma unroll
          for (int b = 0; b < K; ++b) sh_q[a][b] = q[a][b];
        }
        // corner write-back (sparse.hpp:408-429): M(idx[pos], idx[a]) = N(pos, a)
#pragma unroll
        for (int a = 0; a < K; ++a)
#pragma unroll
          for (int p = 0; p < K; ++p) {
            G[static_cast<i64>(loc[a]) * c + loc[p]] = ng[p][a];
            D[static_cast<i64>(loc[a]) * c + loc[p]] = nd[p][a];
          }
#pragma unroll
        for (int a = 0; a < K; ++a) {
          gd[loc[a]] = ng[a][a];
          dd[loc[a]] = nd[a][a];
        }
        const i64 slot = base + nrot;
        int lvl = 0;
        if (!is_exact_identity_k<K>(q)) {
#pragma unroll
          for (int a = 0; a < K; ++a) lvl = max(lvl, level[loc[a]]);
          ++lvl;
#pragma unroll
          for (int a = 0; a < K; ++a) level[loc[a]] = lvl;
        }
        A.rot_level[slot] = lvl;
#pragma unroll
        for (int a = 0; a < K; ++a) {
          A.rot_loc[slot * K + a] = loc[a];
#pragma unroll
          for (int b = 0; b < K; ++b) A.rot_q[(slot * K + a) * K + b] = q[a][b];
        }
        sh_victim = victim;
        A.elim_loc[base + nelim] = victim;
        // old timestamps of the rotated columns for the row pass below; the
        // rotated columns become authoritative for every row
#pragma unroll
        for (int a = 0; a < K; ++a) {
          sh_oldts[a] = ts[loc[a]];
          ts[loc[a]] = nrot + 1;
        }
      }
    }
    __syncthreads();
    TMARK(2)
    // Other warps may still have been reading the bitmask (partner fill)
    // before barrier 2; retire the victim only now.
    if (tid == 0) {
      bits[sh_victim >> 5] &= ~(1u << (sh_victim & 31));
      gcnt[(sh_victim >> 10) & 31] -= 1;
    }
    // ---- off-corner rows of G and D (sparse.hpp:398-439)
    {
      double q[K][K];
#pragma unroll
      for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = 0; b < K; ++b) q[a][b] = sh_q[a][b];
      // kRows rows per thread per round: all column loads are issued before
      // any store, so a round costs one memory round trip.
      constexpr int kRows = (K <= 3) ? 4 : 2;
      int oldts[K];
#pragma unroll
      for (int b = 0; b < K; ++b) oldts[b] = sh_oldts[b];
      for (int r0 = tid; r0 < c; r0 += kRows * kSearchThreads) {
        double vg[kRows][K], vd[kRows][K];
        bool ok[kRows];
#pragma unroll
        for (int j = 0; j < kRows; ++j) {
          const int r = r0 + j * kSearchThreads;
          // Rows of retired indices are never read again by any decision
          // (partners, corners and victims involve active indices only).
          bool skip = r >= c || !is_on(bits, r);
#pragma unroll
          for (int a = 0; a < K; ++a) skip |= loc[a] == r;
          ok[j] = !skip;
          const int tr = ok[j] ? ts[r] : 0;
#pragma unroll
          for (int b = 0; b < K; ++b) {
            const i64 at = tr > oldts[b] ? static_cast<i64>(r) * c + loc[b] : static_cast<i64>(loc[b]) * c + r;
            vg[j][b] = ok[j] ? G[at] : 0.0;
            vd[j][b] = ok[j] ? D[at] : 0.0;
          }
        }
#pragma unroll
        for (int j = 0; j < kRows; ++j) {
          if (!ok[j]) continue;
          const int r = r0 + j * kSearchThreads;
#pragma unroll
          for (int a = 0; a < K; ++a) {
            double ag = 0.0, ad = 0.0;
#pragma unroll
            for (int b = 0; b < K; ++b) {
              ag = dadd(ag, dmul(q[a][b], vg[j][b]));
              ad = dadd(ad, dmul(q[a][b], vd[j][b]));
            }
            G[static_cast<i64>(loc[a]) * c + r] = ag;
            D[static_cast<i64>(loc[a]) * c + r] = ad;
          }
        }
      }
    }
    TMARK(3)
    --count;
    ++nrot;
    ++nelim;
    __syncthreads();
    TMARK(4)
  }
  if (A.timing && tid == 0)
    for (int i = 0; i < 6; ++i) A.timing[static_cast<i64>(u) * 8 + i] = tacc[i];
#undef TMARK
  if (tid == 0) {
    A.nrot[u] = nrot;
    A.nelim[u] = nelim;
  }
}

// ---- large clusters: one thread-block cluster of `csize` CTAs per cluster.
// The per-iteration work (partner scan and off-corner update, both O(c)) is
// split by row slices [lo, hi) across the CTAs, which otherwise run the
// identical iteration: every CTA advances the same RNG stream, keeps full
// copies of the bitmask, diagonals and timestamps, and computes the same
// rotation from the same corner; only rank 0 writes the corner and the
// records.  Per partner round the CTAs exchange their best (score, index)
// through distributed shared memory and reduce it in the same total order
// (strict >, ties to the lowest index), so every decision equals the
// single-CTA kernel's.  G/D are read with ld.global.cg (L2): rows of one
// CTA's slice are written by it, corners by rank 0, and a cluster barrier
// (release/acquire at cluster scope) ends every iteration.
constexpr int kMaxClusterCtas = 16;

template <int K>
__global__ void __launch_bounds__(kSearchThreads, 1) k_search_cl(KArgs A, const int32_t* big_order) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ unsigned char smem[];
  __shared__ Best red[2][kWarps];
  __shared__ Best cand[2][kMaxClusterCtas];
  __shared__ int sh_loc[K];
  __shared__ double sh_q[K][K];
  __shared__ int sh_victim;
  __shared__ int sh_oldts[K];
  const int crank = static_cast<int>(cl.block_rank());
  const int csize = static_cast<int>(cl.num_blocks());
  const int u = big_order[blockIdx.x / csize];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int c = static_cast<int>(A.c[u]);
  if (c < K) {  // uniform over the cluster's CTAs
    if (crank == 0 && tid == 0) {
      A.nrot[u] = 0;
      A.nelim[u] = 0;
    }
    return;
  }
  const i64 base = A.out_base[u];
  i64 budget = static_cast<i64>(floor(A.eta * static_cast<double>(c)));
  if (A.budget[u] >= 0) budget = min(budget, A.budget[u]);
  const int nwords = (c + 31) / 32;
  const int lo = static_cast<int>((static_cast<i64>(c) * crank) / csize);
  const int hi = static_cast<int>((static_cast<i64>(c) * (crank + 1)) / csize);
  uint32_t* bits = reinterpret_cast<uint32_t*>(smem);
  double* gd = reinterpret_cast<double*>(smem + ((static_cast<size_t>(nwords) * 4 + 15) / 16) * 16);
  double* dd = gd + c;
  int32_t* ts = reinterpret_cast<int32_t*>(dd + c);
  int32_t* level = A.level_scratch + static_cast<i64>(u) * A.max_c;
  double* G = A.G + A.tile[u];
  double* D = A.D + A.tile[u];
  __shared__ int gcnt[32];
  const bool sel2 = nwords <= 1024;
  for (int w = tid; w < nwords; w += kSearchThreads) {
    const int h = min(32, c - w * 32);
    bits[w] = h == 32 ? 0xffffffffu : ((1u << h) - 1u);
  }
  if (tid < 32) gcnt[tid] = max(0, min(1024, c - tid * 1024));
  for (int l = tid; l < c; l += kSearchThreads) {
    gd[l] = __ldcg(G + static_cast<i64>(l) * c + l);
    dd[l] = __ldcg(D + static_cast<i64>(l) * c + l);
    ts[l] = 0;
    if (crank == 0) level[l] = 0;
  }
  Xoshiro rng(A.seed[u]);
  int count = c, nrot = 0, nelim = 0, par = 0, cpar = 0;
  unsigned long long tacc[6] = {0, 0, 0, 0, 0, 0}, tprev = clock64();
  const bool timed = A.timing && crank == 0 && tid == 0;
#define CMARK(i)                               \
  if (timed) {                                 \
    const unsigned long long now_ = clock64(); \
    tacc[i] += now_ - tprev;                   \
    tprev = now_;                              \
  }
  cl.sync();

  for (i64 s = 0; s < budget; ++s) {
    if (count <= K - 1) break;
    const int idx = static_cast<int>(rng.uniform_below(static_cast<uint64_t>(count)));
    const int draw = sel2 ? warp_select2(bits, gcnt, nwords, idx) : warp_select(bits, nwords, idx);
    CMARK(0)
    if (gd[draw] <= 0.0) {  // vanished column (:234-238)
      __syncthreads();
      if (tid == 0) {
        bits[draw >> 5] &= ~(1u << (draw & 31));
        gcnt[(draw >> 10) & 31] -= 1;
        if (crank == 0) A.elim_loc[base + nelim] = draw;
      }
      --count;
      ++nelim;
      __syncthreads();
      continue;
    }
    int loc[K];
    loc[0] = draw;
    int npart = 0;
    const double* gcol = G + static_cast<i64>(draw) * c;
    const int tsd = ts[draw];
#pragma unroll 1
    for (int round = 0; round < K - 1; ++round) {
      double bs = 0.0;
      int bl = INT_MAX;
      for (int l0 = lo + tid; l0 < hi; l0 += 2 * kSearchThreads) {
        double gv[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int l = l0 + j * kSearchThreads;
          gv[j] = 0.0;
          if (l < hi && is_on(bits, l))
            gv[j] = ts[l] > tsd ? __ldcg(G + static_cast<i64>(l) * c + draw) : __ldcg(gcol + l);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int l = l0 + j * kSearchThreads;
          if (l >= hi || l == draw || !is_on(bits, l)) continue;
          const double nl = gd[l];
          if (nl <= 0.0) continue;
          bool taken = false;
#pragma unroll
          for (int t = 1; t < K; ++t) taken |= (t <= round) && loc[t] == l;
          if (taken) continue;
          const double sc = (gv[j] * gv[j]) / nl;
          if (sc > 0.0 && better(sc, l, bs, bl)) {
            bs = sc;
            bl = l;
          }
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, bs, o);
        const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
        if (better(os, ol, bs, bl)) {
          bs = os;
          bl = ol;
        }
      }
      if (lane == 0) red[par][wid] = Best{bs, bl};
      __syncthreads();
      if (wid == 0) {
        // CTA best, then published to every CTA of the cluster
        Best b = red[par][0];
        for (int w = 1; w < kWarps; ++w)
          if (better(red[par][w].s, red[par][w].l, b.s, b.l)) b = red[par][w];
        if (lane < csize) {
          Best* dst = cl.map_shared_rank(&cand[cpar][crank], lane);
          *dst = b;
        }
      }
      par ^= 1;
      CMARK(1)
      cl.sync();
      CMARK(2)
      Best b = cand[cpar][0];
      for (int r = 1; r < csize; ++r)
        if (better(cand[cpar][r].s, cand[cpar][r].l, b.s, b.l)) b = cand[cpar][r];
      cpar ^= 1;
      if (!(b.s > 0.0)) break;
#pragma unroll
      for (int t = 1; t < K; ++t)
        if (t == round + 1) loc[t] = b.l;
      ++npart;
    }
    if (npart < K - 1) {
      int have = npart;
      for (int i = 0; have < K - 1; ++i) {
        const int l = sel2 ? warp_select2(bits, gcnt, nwords, i) : warp_select(bits, nwords, i);
        bool taken = l == draw;
#pragma unroll
        for (int t = 1; t < K; ++t) taken |= (t <= have) && loc[t] == l;
        if (!taken) {
#pragma unroll
          for (int t = 1; t < K; ++t)
            if (t == have + 1) loc[t] = l;
          ++have;
        }
      }
    }
    double gs[K][K], cd[K][K];
    if (wid == 0) {
#pragma unroll
      for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = 0; b < K; ++b) {
          const bool rowcol = ts[loc[a]] > ts[loc[b]];
          const i64 at = rowcol ? static_cast<i64>(loc[a]) * c + loc[b] : static_cast<i64>(loc[b]) * c + loc[a];
          gs[a][b] = __ldcg(G + at);
          cd[a][b] = __ldcg(D + at);
        }
    }
    // every CTA has read the corner before rank 0 overwrites it below (a
    // late CTA would otherwise read the NEW corner, derive another rotation
    // for its row slice and leave G asymmetric: the rare "input not
    // symmetric" failures of full-size runs)
    cl.sync();
    if (wid == 0) {
      double q[K][K], ng[K][K], nd[K][K];
      const bool ok = rotation_from_gram_k<K>(gs, q);
      conjugate_corner_k<K>(q, gs, ng);
      conjugate_corner_k<K>(q, cd, nd);
      int victim = -1;
      double vn = 0.0;
#pragma unroll
      for (int a = 1; a < K; ++a) {
        const double off = off_diag_norm_sq(ng[a][a], nd[a][a]);
        if (victim < 0 || off < vn) {
          victim = loc[a];
          vn = off;
        }
      }
      if (off_diag_norm_sq(ng[0][0], nd[0][0]) < vn) victim = draw;
      if (lane == 0) {
#pragma unroll
        for (int a = 0; a < K; ++a) {
          sh_loc[a] = loc[a];
#pragma unroll
          for (int b = 0; b < K; ++b) sh_q[a][b] = q[a][b];
        }
        if (crank == 0) {
          if (!ok) atomicExch(A.error, 1);
#pragma unroll
          for (int a = 0; a < K; ++a)
#pragma unroll
            for (int p = 0; p < K; ++p) {
              G[static_cast<i64>(loc[a]) * c + loc[p]] = ng[p][a];
              D[static_cast<i64>(loc[a]) * c + loc[p]] = nd[p][a];
            }
          const i64 slot = base + nrot;
          int lvl = 0;
          if (!is_exact_identity_k<K>(q)) {
#pragma unroll
            for (int a = 0; a < K; ++a) lvl = max(lvl, level[loc[a]]);
            ++lvl;
#pragma unroll
            for (int a = 0; a < K; ++a) level[loc[a]] = lvl;
          }
          A.rot_level[slot] = lvl;
#pragma unroll
          for (int a = 0; a < K; ++a) {
            A.rot_loc[slot * K + a] = loc[a];
#pragma unroll
            for (int b = 0; b < K; ++b) A.rot_q[(slot * K + a) * K + b] = q[a][b];
          }
          A.elim_loc[base + nelim] = victim;
        }
#pragma unroll
        for (int a = 0; a < K; ++a) {
          gd[loc[a]] = ng[a][a];
          dd[loc[a]] = nd[a][a];
        }
        sh_victim = victim;
#pragma unroll
        for (int a = 0; a < K; ++a) {
          sh_oldts[a] = ts[loc[a]];
          ts[loc[a]] = nrot + 1;
        }
      }
    }
    __syncthreads();
    CMARK(3)
    if (tid == 0) {
      bits[sh_victim >> 5] &= ~(1u << (sh_victim & 31));
      gcnt[(sh_victim >> 10) & 31] -= 1;
    }
    {
      double q[K][K];
#pragma unroll
      for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = 0; b < K; ++b) q[a][b] = sh_q[a][b];
      int oldts[K];
#pragma unroll
      for (int b = 0; b < K; ++b) oldts[b] = sh_oldts[b];
      for (int r = lo + tid; r < hi; r += kSearchThreads) {
        bool skip = !is_on(bits, r);
#pragma unroll
        for (int a = 0; a < K; ++a) skip |= loc[a] == r;
        if (skip) continue;
        const int tr = ts[r];
        double vg[K], vd[K];
#pragma unroll
        for (int b = 0; b < K; ++b) {
          const i64 at = tr > oldts[b] ? static_cast<i64>(r) * c + loc[b] : static_cast<i64>(loc[b]) * c + r;
          vg[b] = __ldcg(G + at);
          vd[b] = __ldcg(D + at);
        }
#pragma unroll
        for (int a = 0; a < K; ++a) {
          double ag = 0.0, ad = 0.0;
#pragma unroll
          for (int b = 0; b < K; ++b) {
            ag = dadd(ag, dmul(q[a][b], vg[b]));
            ad = dadd(ad, dmul(q[a][b], vd[b]));
          }
          G[static_cast<i64>(loc[a]) * c + r] = ag;
          D[static_cast<i64>(loc[a]) * c + r] = ad;
        }
      }
    }
    --count;
    ++nrot;
    ++nelim;
    CMARK(4)
    __threadfence();
    cl.sync();
    CMARK(5)
  }
  if (timed)
    for (int i = 0; i < 6; ++i) A.timing[static_cast<i64>(u) * 8 + i] = tacc[i];
#undef CMARK
  if (crank == 0 && tid == 0) {
    A.nrot[u] = nrot;
    A.nelim[u] = nelim;
  }
}

template <int K>
void launch_cl(const KArgs& a, const int32_t* big_order, i64 nbig, int csize, size_t smem, cudaStream_t s) {
  auto kern = k_search_cl<K>;
  PMMF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  if (csize > 8) PMMF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(nbig * csize));
  cfg.blockDim = dim3(kSearchThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(csize);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  PMMF_CUDA(cudaLaunchKernelEx(&cfg, kern, a, big_order));
  launch_counter().fetch_add(1, std::memory_order_relaxed);
}

// Largest cluster size (16 non-portable, else 8, 4, 2) the device can
// co-schedule for this kernel and shared-memory size.
template <int K>
int cluster_size_for(size_t smem) {
  auto kern = k_search_cl<K>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  (void)cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  (void)cudaGetLastError();
  for (int cs : {16, 8, 4, 2}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(cs));
    cfg.blockDim = dim3(kSearchThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(cs);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n > 0) return cs;
    (void)cudaGetLastError();
  }
  return 0;
}

template <int K>
void launch(const KArgs& a, i64 nclusters, size_t smem, cudaStream_t s) {
  if (smem > 48 * 1024)
    PMMF_CUDA(cudaFuncSetAttribute(k_search<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  PMMF_LAUNCH(k_search<K>, static_cast<unsigned>(nclusters), kSearchThreads, smem, s, a);
}

}  // namespace

void search_clusters(const SearchBatch& b, i64 u0, i64 nclusters, int k, double eta, double* G, double* D,
                     i64 max_c, SearchOut& out, cudaStream_t s) {
  if (nclusters <= 0) return;
  const i64 nwords = (max_c + 31) / 32;
  const size_t bits_bytes = ((static_cast<size_t>(nwords) * 4 + 15) / 16) * 16;
  const size_t diag_bytes = static_cast<size_t>(max_c) * 20;  // gd, dd (fp64) + ts (int32)
  const bool diag_in_smem = bits_bytes + diag_bytes <= 180 * 1024;
  const size_t smem = bits_bytes + (diag_in_smem ? diag_bytes : 0);
  DBuf<double> diag_scratch;
  if (!diag_in_smem) diag_scratch.alloc(nclusters * 3 * max_c, s);
  DBuf<int32_t> level_scratch(nclusters * max_c, s);
  KArgs a{b.c.get(),           b.tile.get(),        b.budget.get(),       b.seed.get(),        b.out_base.get(),
          eta,                 G,                   D,                    diag_scratch.get(),  level_scratch.get(),
          max_c,               diag_in_smem,        out.nrot.get() + u0,  out.nelim.get() + u0, out.rot_loc.get(),
          out.rot_q.get(),     out.rot_level.get(), out.elim_loc.get(),   out.error.get(), nullptr,
          b.order.get()};
  DBuf<unsigned long long> timing;
  const bool tm = std::getenv("PMMF_B200_SEARCH_TIMING") != nullptr;
  if (tm) {
    timing.alloc(nclusters * 8, s);
    timing.zero();
    a.timing = timing.get();
  }
  if (k < 2 || k > 8) fail(PMMF_INVALID_ARGUMENT, "FactorizeParams: k must be in [2, 8]");
  // Large clusters (the sequential critical path of the launch) go to the
  // thread-block-cluster kernel when their full per-CTA state fits in shared
  // memory, with about c/1024 CTAs each (2, 4 or 8: measured best on config
  // 4; a cluster barrier per iteration costs more than wider slices save
  // beyond that); one launch per cluster width, on forked streams alongside
  // the one-CTA kernel.
  i64 big_c = 2048;
  if (const char* e = std::getenv("PMMF_B200_SEARCH_BIG_C")) big_c = std::atoll(e);  // test hook (<= 0: off)
  int cmax = 8, force_w = 0;
  if (const char* e = std::getenv("PMMF_B200_SEARCH_CSIZE")) cmax = std::atoi(e);     // widest cluster
  if (const char* e = std::getenv("PMMF_B200_SEARCH_FORCE_W")) force_w = std::atoi(e);  // test hook
  std::vector<int32_t> h_order = b.order.to_host(nclusters), small;
  std::vector<int32_t> group[5];  // by log2(cluster width)
  size_t gsmem[5] = {0, 0, 0, 0, 0};
  if (big_c > 0 && cmax >= 2 && static_cast<i64>(b.h_c.size()) == nclusters) {
    int dev_max = 0;
    {
      size_t probe = 200 * 1024;
      switch (k) {
        case 2: dev_max = cluster_size_for<2>(probe); break;
        case 3: dev_max = cluster_size_for<3>(probe); break;
        case 4: dev_max = cluster_size_for<4>(probe); break;
        case 5: dev_max = cluster_size_for<5>(probe); break;
        case 6: dev_max = cluster_size_for<6>(probe); break;
        case 7: dev_max = cluster_size_for<7>(probe); break;
        default: dev_max = cluster_size_for<8>(probe); break;
      }
    }
    cmax = std::min(cmax, dev_max);
    auto need_of = [](i64 c) {
      return ((static_cast<size_t>((c + 31) / 32) * 4 + 15) / 16) * 16 + static_cast<size_t>(c) * 20;
    };
    std::vector<int> width(static_cast<size_t>(nclusters), 1);
    for (size_t i = 0; i < h_order.size(); ++i) {
      const int32_t u = h_order[i];
      const i64 c = b.h_c[u];
      int w = 1;
      while (w * 2 <= cmax && static_cast<i64>(w) * 2 * 1024 <= c) w *= 2;
      if (c >= big_c && need_of(c) <= 200 * 1024 && cmax >= 2) {
        w = std::max(w, 2);
        if (force_w >= 2) w = std::min(force_w, cmax);
      } else {
        w = 1;
      }
      width[i] = w;
    }
    // Capacity: the cluster kernel holds one CTA per SM, the single-CTA
    // kernel two.  When the widths ask for more SMs than the device has,
    // the launch runs in waves and wide slices stop paying: narrow the
    // cheapest clusters first (model: c/2 iterations of alpha + beta c/w,
    // measured on config 4: 34 us at c = 8192 on 1 CTA, ~7 us on 8 CTAs)
    // until the summed SM-time fits under the longest cluster's time.
    if (force_w < 2) {
      int nsm = 148;
      {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) (void)cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      }
      // per-iteration cost alpha + beta c / w (us); tunable for the sweep in
      // scripts/search_sweep.sh
      double a1 = 3.0, acl = 3.0, beta = 0.0035;
      if (const char* e = std::getenv("PMMF_B200_SEARCH_A1")) a1 = std::atof(e);
      if (const char* e = std::getenv("PMMF_B200_SEARCH_ACL")) acl = std::atof(e);
      if (const char* e = std::getenv("PMMF_B200_SEARCH_BETA")) beta = std::atof(e);
      auto t_of = [=](i64 c, int w) {
        return 0.5 * static_cast<double>(c) * ((w >= 2 ? acl : a1) + beta * static_cast<double>(c) / w);
      };
      auto sm_time = [&](i64 c, int w) { return (w >= 2 ? w : 0.5) * t_of(c, w); };
      for (;;) {
        double work = 0.0, longest = 0.0;
        for (size_t i = 0; i < h_order.size(); ++i) {
          const i64 c = b.h_c[h_order[i]];
          work += sm_time(c, width[i]);
          longest = std::max(longest, t_of(c, width[i]));
        }
        if (work / nsm <= longest) break;
        // narrow the cluster whose halved time stays smallest
        size_t best = h_order.size();
        double bt = 0.0;
        for (size_t i = 0; i < h_order.size(); ++i) {
          if (width[i] < 2) continue;
          const double t = t_of(b.h_c[h_order[i]], width[i] / 2);
          if (best == h_order.size() || t < bt) {
            best = i;
            bt = t;
          }
        }
        if (best == h_order.size()) break;
        width[best] /= 2;
      }
    }
    for (size_t i = 0; i < h_order.size(); ++i) {
      const int32_t u = h_order[i];
      const int w = width[i];
      if (w >= 2) {
        const int g = w >= 16 ? 4 : w >= 8 ? 3 : w >= 4 ? 2 : 1;
        group[g].push_back(u);
        gsmem[g] = std::max(gsmem[g], need_of(b.h_c[u]));
      } else {
        small.push_back(u);
      }
    }
  } else {
    small = h_order;
  }
  DBuf<int32_t> d_group[5], d_small;
  std::vector<cudaStream_t> side;
  std::vector<cudaEvent_t> joins;
  cudaEvent_t fork = nullptr;
  size_t nbig = 0;
  for (int g = 4; g >= 1; --g) {
    if (group[g].empty()) continue;
    nbig += group[g].size();
    if (!fork) {
      PMMF_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
      PMMF_CUDA(cudaEventRecord(fork, s));
    }
    cudaStream_t s2 = nullptr;
    cudaEvent_t join = nullptr;
    PMMF_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    PMMF_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    PMMF_CUDA(cudaStreamWaitEvent(s2, fork, 0));
    d_group[g].alloc(static_cast<i64>(group[g].size()), s);
    d_group[g].upload(group[g]);
    PMMF_CUDA(cudaEventRecord(join, s));  // upload ordered before the side launch
    PMMF_CUDA(cudaStreamWaitEvent(s2, join, 0));
    const i64 nb = static_cast<i64>(group[g].size());
    const int cs = 1 << g;
    switch (k) {
      case 2: launch_cl<2>(a, d_group[g].get(), nb, cs, gsmem[g], s2); break;
      case 3: launch_cl<3>(a, d_group[g].get(), nb, cs, gsmem[g], s2); break;
      case 4: launch_cl<4>(a, d_group[g].get(), nb, cs, gsmem[g], s2); break;
      case 5: launch_cl<5>(a, d_group[g].get(), nb, cs, gsmem[g], s2); break;
      case 6: launch_cl<6>(a, d_group[g].get(), nb, cs, gsmem[g], s2); break;
      case 7: launch_cl<7>(a, d_group[g].get(), nb, cs, gsmem[g], s2); break;
      default: launch_cl<8>(a, d_group[g].get(), nb, cs, gsmem[g], s2); break;
    }
    PMMF_CUDA(cudaEventRecord(join, s2));
    side.push_back(s2);
    joins.push_back(join);
  }
  if (!small.empty()) {
    KArgs as = a;
    if (nbig > 0) {
      d_small.alloc(static_cast<i64>(small.size()), s);
      d_small.upload(small);
      as.order = d_small.get();
    }
    const i64 ns = static_cast<i64>(small.size());
    switch (k) {
      case 2: launch<2>(as, ns, smem, s); break;
      case 3: launch<3>(as, ns, smem, s); break;
      case 4: launch<4>(as, ns, smem, s); break;
      case 5: launch<5>(as, ns, smem, s); break;
      case 6: launch<6>(as, ns, smem, s); break;
      case 7: launch<7>(as, ns, smem, s); break;
      default: launch<8>(as, ns, smem, s); break;
    }
  }
  for (size_t i = 0; i < side.size(); ++i) {
    PMMF_CUDA(cudaStreamWaitEvent(s, joins[i], 0));
    cudaEventDestroy(joins[i]);
    cudaStreamDestroy(side[i]);  // destruction is deferred until its work completes
  }
  if (fork) cudaEventDestroy(fork);
  // the group buffers are released on s, after the join
  if (trace_enabled())
    std::fprintf(stderr, "[pmmf]   search: %zu/%zu/%zu/%zu clusters on 2/4/8/16-CTA clusters, %zu on single CTAs\n",
                 group[1].size(), group[2].size(), group[3].size(), group[4].size(), small.size());
  if (tm) {
    std::vector<unsigned long long> h = timing.to_host(nclusters * 8);
    unsigned long long tot[6] = {0, 0, 0, 0, 0, 0}, mx = 0;
    i64 arg = 0;
    for (i64 u = 0; u < nclusters; ++u) {
      unsigned long long t = 0;
      for (int i = 0; i < 6; ++i) t += h[u * 8 + i];
      if (t > mx) {
        mx = t;
        arg = u;
      }
    }
    std::vector<int64_t> hc = b.c.to_host(nclusters);
    double sum = 0.0;
    for (i64 u = 0; u < nclusters; ++u)
      for (int i = 0; i < 6; ++i) sum += static_cast<double>(h[u * 8 + i]);
    std::vector<i64> ord(static_cast<size_t>(nclusters));
    std::iota(ord.begin(), ord.end(), i64{0});
    auto tot_of = [&](i64 u) {
      unsigned long long t = 0;
      for (int i = 0; i < 6; ++i) t += h[u * 8 + i];
      return t;
    };
    std::sort(ord.begin(), ord.end(), [&](i64 x, i64 y) { return tot_of(x) > tot_of(y); });
    std::fprintf(stderr, "[pmmf] search timing: %lld clusters, all %.3g cycles; slowest:\n", static_cast<long long>(nclusters), sum);
    for (size_t i = 0; i < std::min<size_t>(5, ord.size()); ++i) {
      const i64 u = ord[i];
      std::fprintf(stderr, "[pmmf]     c=%lld total %llu: %llu %llu %llu %llu %llu %llu\n", static_cast<long long>(hc[u]),
                   tot_of(u), h[u * 8 + 0], h[u * 8 + 1], h[u * 8 + 2], h[u * 8 + 3], h[u * 8 + 4], h[u * 8 + 5]);
    }
    (void)arg;
    (void)mx;
    (void)tot;
  }
}

}  // namespace pmmf_b200
