// apply.cu — the stage apply A <- Q A Q^T (factorizer.hpp:336-394) as
// column rotation streams.
//
// Rotations of one stage are grouped into dependency levels (computed by the
// search kernel): a level's rotations touch pairwise disjoint ids, so they
// run concurrently, one warp per rotation, and levels run in order.  For a
// rotation on ids (j_0..j_k-1) the warp merges the k sorted sparse columns
// window by window (32 rows per list per step), forms
//   out_a = ((0 + q(a,0) v_0) + q(a,1) v_1) + ...            (sparse.hpp:123-156)
// over the union support with absent entries = 0.0, drops exact zeros
// (value-neutral) and appends the k new columns to the
// arena.  The row side is the same kernel on the transpose (App. A P12,
// "transpose trick").  HBM-bound streaming: every input entry is read once
// and every output entry written once per rotation.
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>

#include "engine.cuh"

namespace pmmf_b200 {

namespace {

constexpr int kThreads = 256;

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

template <int K>
__global__ void k_rotate_level(i64 n, const int32_t* __restrict__ order, const int32_t* __restrict__ ids,
                               const double* __restrict__ qs, i64* __restrict__ off, int32_t* __restrict__ len,
                               int32_t* __restrict__ arow, double* __restrict__ aval,
                               unsigned long long* __restrict__ cursor, i64 cap, int32_t* __restrict__ overflow,
                               uint8_t* __restrict__ done) {
  const i64 w = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  if (*reinterpret_cast<volatile int32_t*>(overflow)) return;
  const int t = order[w];
  if (done[t]) return;
  i64 src[K];
  int L[K], p[K];
  int id[K];
  double q[K][K];
  i64 S = 0;
#pragma unroll
  for (int b = 0; b < K; ++b) {
    id[b] = ids[static_cast<i64>(t) * K + b];
    src[b] = off[id[b]];
    L[b] = len[id[b]];
    p[b] = 0;
    S += L[b];
#pragma unroll
    for (int a = 0; a < K; ++a) q[b][a] = qs[(static_cast<i64>(t) * K + b) * K + a];
  }
  unsigned long long base = 0;
  if (lane == 0) {
    base = atomicAdd(cursor, static_cast<unsigned long long>(K) * static_cast<unsigned long long>(S));
    if (static_cast<i64>(base) + K * S > cap) atomicExch(overflow, 1);
  }
  base = __shfl_sync(0xffffffffu, base, 0);
  if (static_cast<i64>(base) + K * S > cap) return;
  int written[K];
#pragma unroll
  for (int a = 0; a < K; ++a) written[a] = 0;

  for (;;) {
    int row[K];
    double val[K];
    int frontier = INT_MAX;
    bool any = false;
#pragma unroll
    for (int b = 0; b < K; ++b) {
      const int e = p[b] + lane;
      row[b] = e < L[b] ? arow[src[b] + e] : INT_MAX;
      val[b] = e < L[b] ? aval[src[b] + e] : 0.0;
      const int last = __shfl_sync(0xffffffffu, row[b], 31);
      frontier = min(frontier, last);
      any |= p[b] < L[b];
    }
    if (!any) break;
    bool valid[K];
    unsigned nvalid[K];
#pragma unroll
    for (int b = 0; b < K; ++b) {
      valid[b] = row[b] != INT_MAX && row[b] <= frontier;
      nvalid[b] = __popc(__ballot_sync(0xffffffffu, valid[b]));
    }
    // lb[b][b2]: rows of window b2 below row[b] (own window: lane)
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
          present[b][b2] = __shfl_sync(0xffffffffu, row[b2], l & 31) == row[b] && l < 32;
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
    // union rank and mixed values of every first occurrence
    int rank[K];
    double out[K][K];  // out[b][a]: output a for the row owned by window b
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
    // zero-drop compaction in union-rank order, per output column
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
#pragma unroll
      for (int b = 0; b < K; ++b) {
        if (first[b] && out[b][a] != 0.0) {
          int pos = 0;
          const int wd = rank[b] >> 5, bit = rank[b] & 31;
#pragma unroll
          for (int x = 0; x < K; ++x)
            if (x < wd) pos += __popc(words[x]);
          pos += __popc(words[wd] & ((1u << bit) - 1u));
          const i64 dst = static_cast<i64>(base) + static_cast<i64>(a) * S + written[a] + pos;
          arow[dst] = row[b];
          aval[dst] = out[b][a];
        }
      }
      written[a] += total;
    }
#pragma unroll
    for (int b = 0; b < K; ++b) p[b] += static_cast<int>(nvalid[b]);
  }
  __syncwarp();
  if (lane == 0) {
#pragma unroll
    for (int a = 0; a < K; ++a) {
      off[id[a]] = static_cast<i64>(base) + static_cast<i64>(a) * S;
      len[id[a]] = written[a];
    }
    done[t] = 1;
  }
}

// Compaction of the live columns into a fresh arena.
__global__ void k_len64(i64 N, const int32_t* __restrict__ len, i64* __restrict__ out) {
  const i64 j = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (j < N) out[j] = len[j];
  if (j == N) out[j] = 0;
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

void compact(Paged& P, i64 min_free, cudaStream_t s) {
  DBuf<i64> l64(P.N + 1, s), pos(P.N + 1, s);
  PMMF_LAUNCH(k_len64, blocks_for(P.N + 1, kThreads), kThreads, 0, s, P.N, P.len.get(), l64.get());
  size_t tmp = 0;
  PMMF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, l64.get(), pos.get(), static_cast<int64_t>(P.N + 1), s));
  DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
  PMMF_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, l64.get(), pos.get(), static_cast<int64_t>(P.N + 1), s));
  i64 live = 0;
  PMMF_CUDA(cudaMemcpyAsync(&live, pos.get() + P.N, sizeof(i64), cudaMemcpyDeviceToHost, s));
  PMMF_CUDA(cudaStreamSynchronize(s));
  const i64 cap = std::max<i64>(2 * live, live + min_free) + 1024;
  DBuf<int32_t> r1(cap, s);
  DBuf<double> v1(cap, s);
  PMMF_LAUNCH(k_compact, blocks_for(P.N * 32, kThreads), kThreads, 0, s, P.N, P.off.get(), P.len.get(), pos.get(),
              P.row.get(), P.val.get(), r1.get(), v1.get());
  P.row = std::move(r1);
  P.val = std::move(v1);
  P.cap = cap;
  const unsigned long long c0 = static_cast<unsigned long long>(live);
  PMMF_CUDA(cudaMemcpyAsync(P.cursor.get(), &c0, sizeof(c0), cudaMemcpyHostToDevice, s));
  PMMF_CUDA(cudaStreamSynchronize(s));
}

template <int K>
void launch_level(Paged& P, const LevelPlan& plan, i64 begin, i64 count, DBuf<int32_t>& overflow,
                  DBuf<uint8_t>& done, cudaStream_t s) {
  PMMF_LAUNCH(k_rotate_level<K>, blocks_for(count * 32, kThreads), kThreads, 0, s, count, plan.order.get() + begin,
              plan.ids.get(), plan.q, P.off.get(), P.len.get(), P.row.get(), P.val.get(), P.cursor.get(), P.cap,
              overflow.get(), done.get());
}

__global__ void k_plan(const int32_t* __restrict__ nrot, const int64_t* __restrict__ base,
                       const int64_t* __restrict__ coff, const int32_t* __restrict__ rot_loc,
                       const int32_t* __restrict__ rot_level, int k, int32_t* __restrict__ ids,
                       int32_t* __restrict__ lvl, int32_t* __restrict__ slot) {
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

void build_plan(LevelPlan& plan, const SearchOut& so, const DBuf<int64_t>& out_base,
                const DBuf<int64_t>& cluster_off, i64 nclusters, i64 R, int k, cudaStream_t s) {
  plan.R = R;
  plan.k = k;
  plan.q = so.rot_q.get();
  plan.max_level = 0;
  plan.level_start.assign(1, 0);
  if (R == 0 || nclusters == 0) return;
  plan.ids.alloc(R * k, s);
  DBuf<int32_t> lvl(R, s), slot(R, s), lvl2(R, s);
  lvl.zero();
  PMMF_LAUNCH(k_plan, static_cast<unsigned>(nclusters), 256, 0, s, so.nrot.get(), out_base.get(), cluster_off.get(),
              so.rot_loc.get(), so.rot_level.get(), k, plan.ids.get(), lvl.get(), slot.get());
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
  // level L (1-based) occupies [h[L], h[L+1]) of the sorted order
  plan.level_start.assign(h.begin() + 1, h.end());
}

void apply_levels(Paged& P, const LevelPlan& plan, cudaStream_t s) {
  if (plan.R == 0 || plan.max_level == 0) return;
  DBuf<int32_t> overflow(1, s);
  DBuf<uint8_t> done(plan.R, s);
  overflow.zero();
  done.zero();
  for (int attempt = 0;; ++attempt) {
    for (int L = 1; L <= plan.max_level; ++L) {
      const i64 b = plan.level_start[L - 1], cnt = plan.level_start[L] - b;
      switch (plan.k) {
        case 2: launch_level<2>(P, plan, b, cnt, overflow, done, s); break;
        case 3: launch_level<3>(P, plan, b, cnt, overflow, done, s); break;
        case 4: launch_level<4>(P, plan, b, cnt, overflow, done, s); break;
        case 5: launch_level<5>(P, plan, b, cnt, overflow, done, s); break;
        case 6: launch_level<6>(P, plan, b, cnt, overflow, done, s); break;
        case 7: launch_level<7>(P, plan, b, cnt, overflow, done, s); break;
        case 8: launch_level<8>(P, plan, b, cnt, overflow, done, s); break;
        default: fail(PMMF_INVALID_ARGUMENT, "apply: unsupported k");
      }
    }
    int32_t of = 0;
    PMMF_CUDA(cudaMemcpyAsync(&of, overflow.get(), sizeof(of), cudaMemcpyDeviceToHost, s));
    PMMF_CUDA(cudaStreamSynchronize(s));
    if (!of) return;
    if (attempt > 40) fail(PMMF_INTERNAL, "apply: arena compaction did not converge");
    compact(P, P.cap, s);  // at least double the free space
    overflow.zero();
  }
}

}  // namespace pmmf_b200
