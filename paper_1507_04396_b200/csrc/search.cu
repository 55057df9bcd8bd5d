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
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>

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
  for (int w = tid; w < nwords; w += kSearchThreads) {
    const int hi = min(32, c - w * 32);
    bits[w] = hi == 32 ? 0xffffffffu : ((1u << hi) - 1u);
  }
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
    const int draw = warp_select(bits, nwords, idx);
    TMARK(0)
    if (gd[draw] <= 0.0) {  // vanished column: retire without a rotation (:234-238)
      __syncthreads();      // everyone has read bits for this draw
      if (tid == 0) {
        bits[draw >> 5] &= ~(1u << (draw & 31));
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
        const int l = warp_select(bits, nwords, i);
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
    if (tid == 0) bits[sh_victim >> 5] &= ~(1u << (sh_victim & 31));
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
  switch (k) {
    case 2: launch<2>(a, nclusters, smem, s); break;
    case 3: launch<3>(a, nclusters, smem, s); break;
    case 4: launch<4>(a, nclusters, smem, s); break;
    case 5: launch<5>(a, nclusters, smem, s); break;
    case 6: launch<6>(a, nclusters, smem, s); break;
    case 7: launch<7>(a, nclusters, smem, s); break;
    case 8: launch<8>(a, nclusters, smem, s); break;
    default: fail(PMMF_INVALID_ARGUMENT, "FactorizeParams: k must be in [2, 8]");
  }
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
    std::fprintf(stderr, "[pmmf] search timing (slowest cluster %lld of %lld): select %llu partner %llu rot %llu offcorner %llu barrier %llu cycles\n",
                 static_cast<long long>(arg), static_cast<long long>(nclusters), h[arg * 8 + 0], h[arg * 8 + 1],
                 h[arg * 8 + 2], h[arg * 8 + 3], h[arg * 8 + 4]);
  }
}

}  // namespace pmmf_b200
