// search.cu — randomized greedy k-tuple pivot search (Algorithm 2,
// factorizer.hpp:198-319), one CTA per cluster, all clusters of a stage in
// one launch.
//
// Per cluster the state is the dense column-major Gram tile G_u and diagonal
// block D_u (full storage: the conjugated k x k corner is not bitwise
// symmetric), the active set as a bitmask in shared
// memory, and the diagonals of G and D in shared memory.  Each iteration:
//   1. lane 0 draws uniform_below(|active|) from the cluster's stream
//      (P5); warp 0 selects the idx-th active index with popc prefix sums;
//   2. the CTA scans column `draw` of G for the best partner(s)
//      (score g^2 / G_ll, strict >, ties to the lowest index; P8);
//   3. one thread builds q = rotation_from_gram (P9) and the conjugated
//      corners of G and D;
//   4. the CTA rewrites the k columns and k mirrored rows of G and D over
//      every off-corner row (P10), coalesced on the column side;
//   5. one thread picks the victim (P11), retires it and records the
//      rotation with its dependency level for the stage apply.
// Everything is exact fp64 without contraction (-fmad=false).
#include <algorithm>
#include <climits>

#include "engine.cuh"
#include "rng.cuh"
#include "rotation.cuh"

namespace pmmf_b200 {

namespace {

constexpr int kSearchThreads = 256;
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
  int k;
  double eta;
  double* G;
  double* D;
  double* diag_scratch;   // 2 * max_c per cluster when the diagonals do not fit in shared memory
  int32_t* level_scratch; // max_c per cluster
  i64 max_c;
  bool diag_in_smem;
  int32_t* nrot;
  int32_t* nelim;
  int32_t* rot_loc;
  double* rot_q;
  int32_t* rot_level;
  int32_t* elim_loc;
  int32_t* error;
};

__global__ void __launch_bounds__(kSearchThreads) k_search(KArgs A) {
  extern __shared__ unsigned char smem[];
  __shared__ Best red[kWarps];
  __shared__ int sh_draw, sh_stop, sh_idx, sh_count, sh_npart;
  __shared__ int sh_loc[kMaxK];
  __shared__ double sh_q[kMaxK][kMaxK];
  const int u = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const i64 c64 = A.c[u];
  const int k = A.k;
  const i64 base = A.out_base[u];
  if (c64 < k) {
    if (tid == 0) {
      A.nrot[u] = 0;
      A.nelim[u] = 0;
    }
    return;
  }
  const int c = static_cast<int>(c64);
  i64 budget = static_cast<i64>(floor(A.eta * static_cast<double>(c)));
  if (A.budget[u] >= 0) budget = min(budget, A.budget[u]);
  const int nwords = (c + 31) / 32;
  uint32_t* bits = reinterpret_cast<uint32_t*>(smem);
  double* gd;
  double* dd;
  if (A.diag_in_smem) {
    gd = reinterpret_cast<double*>(smem + ((static_cast<size_t>(nwords) * 4 + 15) / 16) * 16);
    dd = gd + c;
  } else {
    gd = A.diag_scratch + static_cast<i64>(u) * 2 * A.max_c;
    dd = gd + c;
  }
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
    level[l] = 0;
  }
  if (tid == 0) sh_count = c;
  Xoshiro rng(A.seed[u]);  // meaningful in thread 0 only
  int nrot = 0, nelim = 0;
  __syncthreads();

  for (i64 s = 0; s < budget; ++s) {
    if (tid == 0) {
      sh_stop = sh_count <= k - 1;
      if (!sh_stop) sh_idx = static_cast<int>(rng.uniform_below(static_cast<uint64_t>(sh_count)));
    }
    __syncthreads();
    if (sh_stop) break;
    if (wid == 0) {
      const int d = warp_select(bits, nwords, sh_idx);
      if (lane == 0) sh_draw = d;
    }
    __syncthreads();
    const int draw = sh_draw;
    if (gd[draw] <= 0.0) {  // vanished column: retire without a rotation (:234-238)
      if (tid == 0) {
        bits[draw >> 5] &= ~(1u << (draw & 31));
        --sh_count;
        A.elim_loc[base + nelim] = draw;
      }
      ++nelim;
      __syncthreads();
      continue;
    }
    // ---- partners (:243-280)
    const double* gcol = G + static_cast<i64>(draw) * c;
    if (tid == 0) {
      sh_loc[0] = draw;
      sh_npart = 0;
    }
    __syncthreads();
    for (int round = 0; round < k - 1; ++round) {
      double bs = 0.0;
      int bl = INT_MAX;
      for (int l = tid; l < c; l += kSearchThreads) {
        if (l == draw || !is_on(bits, l)) continue;
        const double nl = gd[l];
        if (nl <= 0.0) continue;
        bool taken = false;
        for (int t = 1; t <= round; ++t) taken |= sh_loc[t] == l;
        if (taken) continue;
        const double g = gcol[l];
        const double sc = (g * g) / nl;
        if (sc > 0.0 && better(sc, l, bs, bl)) {
          bs = sc;
          bl = l;
        }
      }
      for (int o = 16; o; o >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, bs, o);
        const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
        if (better(os, ol, bs, bl)) {
          bs = os;
          bl = ol;
        }
      }
      if (lane == 0) red[wid] = Best{bs, bl};
      __syncthreads();
      if (tid == 0) {
        Best b = red[0];
        for (int w = 1; w < kWarps; ++w)
          if (better(red[w].s, red[w].l, b.s, b.l)) b = red[w];
        if (b.s > 0.0) {
          sh_loc[1 + round] = b.l;
          sh_npart = round + 1;
        }
      }
      __syncthreads();
      if (sh_npart != round + 1) break;  // no more positive scores
    }
    if (sh_npart < k - 1 && wid == 0) {
      // Fill with the lowest active indices not yet chosen (:256, :275-279).
      int have = sh_npart;
      for (int idx = 0; have < k - 1; ++idx) {
        const int l = warp_select(bits, nwords, idx);
        bool taken = l == draw;
        for (int t = 1; t <= have; ++t) taken |= sh_loc[t] == l;
        if (!taken) {
          if (lane == 0) sh_loc[1 + have] = l;
          ++have;
        }
        __syncwarp();
      }
      if (lane == 0) sh_npart = have;
    }
    __syncthreads();
    // ---- rotation (:287-298) and the k x k corners
    if (tid == 0) {
      double gs[kMaxK][kMaxK], cd[kMaxK][kMaxK], q[kMaxK][kMaxK], ng[kMaxK][kMaxK], nd[kMaxK][kMaxK];
      for (int a = 0; a < k; ++a)
        for (int b = 0; b < k; ++b) {
          gs[a][b] = G[static_cast<i64>(sh_loc[b]) * c + sh_loc[a]];
          cd[a][b] = D[static_cast<i64>(sh_loc[b]) * c + sh_loc[a]];
        }
      if (!rotation_from_gram(gs, k, q)) atomicExch(A.error, 1);
      conjugate_corner(q, gs, k, ng);
      conjugate_corner(q, cd, k, nd);
      for (int a = 0; a < k; ++a)
        for (int b = 0; b < k; ++b) sh_q[a][b] = q[a][b];
      // corner write-back (sparse.hpp:408-429): M(idx[pos], idx[a]) = N(pos, a)
      for (int a = 0; a < k; ++a)
        for (int p = 0; p < k; ++p) {
          G[static_cast<i64>(sh_loc[a]) * c + sh_loc[p]] = ng[p][a];
          D[static_cast<i64>(sh_loc[a]) * c + sh_loc[p]] = nd[p][a];
        }
      for (int a = 0; a < k; ++a) {
        gd[sh_loc[a]] = ng[a][a];
        dd[sh_loc[a]] = nd[a][a];
      }
      // victim (:300-316)
      int victim = -1;
      double vn = 0.0;
      for (int a = 1; a < k; ++a) {
        const int l = sh_loc[a];
        const double off = off_diag_norm_sq(gd[l], dd[l]);
        if (victim < 0 || off < vn) {
          victim = l;
          vn = off;
        }
      }
      if (off_diag_norm_sq(gd[draw], dd[draw]) < vn) victim = draw;
      // record + dependency level for the stage apply
      const i64 slot = base + nrot;
      int lvl = 0;
      if (!is_exact_identity(q, k)) {
        for (int a = 0; a < k; ++a) lvl = max(lvl, level[sh_loc[a]]);
        ++lvl;
        for (int a = 0; a < k; ++a) level[sh_loc[a]] = lvl;
      }
      A.rot_level[slot] = lvl;
      for (int a = 0; a < k; ++a) {
        A.rot_loc[slot * k + a] = sh_loc[a];
        for (int b = 0; b < k; ++b) A.rot_q[(slot * k + a) * k + b] = q[a][b];
      }
      bits[victim >> 5] &= ~(1u << (victim & 31));
      --sh_count;
      A.elim_loc[base + nelim] = victim;
    }
    __syncthreads();
    // ---- off-corner rows of G and D (sparse.hpp:398-439)
    {
      int loc[kMaxK];
      double q[kMaxK][kMaxK];
      for (int a = 0; a < k; ++a) {
        loc[a] = sh_loc[a];
        for (int b = 0; b < k; ++b) q[a][b] = sh_q[a][b];
      }
      for (int r = tid; r < c; r += kSearchThreads) {
        bool corner = false;
        for (int a = 0; a < k; ++a) corner |= loc[a] == r;
        if (corner) continue;
#pragma unroll 1
        for (int mtx = 0; mtx < 2; ++mtx) {
          double* M = mtx ? D : G;
          double v[kMaxK], mixed[kMaxK];
          for (int b = 0; b < k; ++b) v[b] = M[static_cast<i64>(loc[b]) * c + r];
          for (int a = 0; a < k; ++a) {
            double acc = 0.0;
            for (int b = 0; b < k; ++b) acc = dadd(acc, dmul(q[a][b], v[b]));
            mixed[a] = acc;
          }
          for (int a = 0; a < k; ++a) {
            M[static_cast<i64>(loc[a]) * c + r] = mixed[a];
            M[static_cast<i64>(r) * c + loc[a]] = mixed[a];
          }
        }
      }
    }
    ++nrot;
    ++nelim;
    __syncthreads();
  }
  if (tid == 0) {
    A.nrot[u] = nrot;
    A.nelim[u] = nelim;
  }
}

}  // namespace

void search_clusters(const SearchBatch& b, i64 u0, i64 nclusters, int k, double eta, double* G, double* D,
                     i64 max_c, SearchOut& out, cudaStream_t s) {
  if (nclusters <= 0) return;
  const i64 nwords = (max_c + 31) / 32;
  const size_t bits_bytes = ((static_cast<size_t>(nwords) * 4 + 15) / 16) * 16;
  const size_t diag_bytes = static_cast<size_t>(max_c) * 16;
  const bool diag_in_smem = bits_bytes + diag_bytes <= 160 * 1024;
  const size_t smem = bits_bytes + (diag_in_smem ? diag_bytes : 0);
  DBuf<double> diag_scratch;
  if (!diag_in_smem) diag_scratch.alloc(nclusters * 2 * max_c, s);
  DBuf<int32_t> level_scratch(nclusters * max_c, s);
  if (smem > 48 * 1024)
    PMMF_CUDA(cudaFuncSetAttribute(k_search, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  KArgs a{b.c.get(),        b.tile.get(),         b.budget.get(),    b.seed.get(),      b.out_base.get(),
          k,                eta,                  G,                 D,                 diag_scratch.get(),
          level_scratch.get(), max_c,             diag_in_smem,      out.nrot.get() + u0, out.nelim.get() + u0,
          out.rot_loc.get(), out.rot_q.get(),     out.rot_level.get(), out.elim_loc.get(), out.error.get()};
  PMMF_LAUNCH(k_search, static_cast<unsigned>(nclusters), kSearchThreads, smem, s, a);
}

}  // namespace pmmf_b200
