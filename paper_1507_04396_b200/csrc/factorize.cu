// factorize.cu — the stage loop of pmmf::factorize (factorizer.hpp:397-595)
// driving the device kernels, plus the result half of the C-ABI.
//
// Per stage p (all matrix data stays in HBM):
//   cluster (cluster.cu, on the PRE-reblock matrix, factorizer.hpp:437)
//   -> reblock into stage numbering (matrix.cu, :456)
//   -> budgets (host, :463-479)
//   -> Gram + diagonal tiles (gram.cu, :485-488) -> search (search.cu, :494-504)
//   -> apply: column pass, transpose, column pass, transpose (apply.cu, :513)
//   -> residual / retired diagonals (k_residual, :521-547) -> shrink (:550-557)
// The host keeps only what the reference keeps on its control path: the
// active list, the partitions, the RNG stream of the clustering, and the
// materialised outputs (rotations, eliminations).
#include <algorithm>
#include <future>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>

#include "engine.cuh"
#include "result.cuh"
#include "rng.cuh"
#include "rotation.cuh"
#include "shard.cuh"

namespace pmmf_b200 {

namespace {

constexpr int kThreads = 256;

// Residual accounting for the stage's eliminations in order r
// (factorizer.hpp:529-542): mass = sum of v^2 over column g's entries whose
// row is still active or retired later in the stage; diag = A'[g][g].
__device__ __forceinline__ void residual_column(i64 r, int32_t j, const int32_t* __restrict__ row,
                                                const double* __restrict__ val, i64 b, i64 e,
                                                const int32_t* __restrict__ s2g, const uint8_t* __restrict__ is_active,
                                                const int32_t* __restrict__ rank, double* __restrict__ mass,
                                                double* __restrict__ diag) {
  // warp: lanes classify 32 entries at a time, lane 0 accumulates them in
  // row order (sequential sum, as the reference does)
  const int lane = threadIdx.x & 31;
  double m = 0.0, d = 0.0;
  for (i64 x = b; x < e; x += 32) {
    const i64 i = x + lane;
    double sq = 0.0;
    bool take = false, isdiag = false;
    double v = 0.0;
    if (i < e) {
      const int32_t sr = row[i];
      v = val[i];
      if (sr == j) {
        isdiag = true;
      } else {
        const int32_t l = s2g[sr];
        take = is_active[l] || rank[l] > r;
        sq = dmul(v, v);
      }
    }
    const unsigned tk = __ballot_sync(0xffffffffu, take);
    const unsigned dg = __ballot_sync(0xffffffffu, isdiag);
    if (dg) d = __shfl_sync(0xffffffffu, v, __ffs(dg) - 1);
    for (unsigned mm = tk; mm; mm &= mm - 1) {
      const int src = __ffs(mm) - 1;
      m = dadd(m, __shfl_sync(0xffffffffu, sq, src));
    }
  }
  if (lane == 0) {
    mass[r] = m;
    diag[r] = d;
  }
}

// Residual accounting for the stage's eliminations in order r
// (factorizer.hpp:529-542): mass = sum of v^2 over column g's entries whose
// row is still active or retired later in the stage; diag = A'[g][g].
__global__ void k_residual(i64 R, const int32_t* __restrict__ elim_sid, const i64* __restrict__ ptr,
                           const int32_t* __restrict__ row, const double* __restrict__ val,
                           const int32_t* __restrict__ s2g, const uint8_t* __restrict__ is_active,
                           const int32_t* __restrict__ rank, double* __restrict__ mass, double* __restrict__ diag,
                           i64 c0, i64 c1) {
  const i64 r = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  if (r >= R) return;
  const int32_t j = elim_sid[r];
  if (j < c0 || j >= c1) return;  // another rank's column
  residual_column(r, j, row, val, ptr[j], ptr[j + 1], s2g, is_active, rank, mass, diag);
}

__global__ void k_mark(i64 R, const int32_t* __restrict__ g, uint8_t* __restrict__ is_active,
                       int32_t* __restrict__ rank, int set_rank) {
  const i64 r = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (r >= R) return;
  is_active[g[r]] = 0;
  rank[g[r]] = set_rank ? static_cast<int32_t>(r) : -1;
}

// Residual keys by stage id: the rank of a retired id (row_rank, else -1)
// and the column key (its rank, or 0x7f7f7f7f for a survivor).
__global__ void k_mass_keys(i64 R, const int32_t* __restrict__ sid, int32_t* __restrict__ row_rank,
                            int32_t* __restrict__ col_key) {
  const i64 r = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (r >= R) return;
  row_rank[sid[r]] = static_cast<int32_t>(r);
  col_key[sid[r]] = static_cast<int32_t>(r);
}

// Core: core(a, b) = A[active[a]][active[b]] (factorizer.hpp:578-588).
__global__ void k_core(i64 g, const int32_t* __restrict__ col_sid, const i64* __restrict__ ptr,
                       const int32_t* __restrict__ row, const double* __restrict__ val,
                       const int32_t* __restrict__ pos_of_sid, double* __restrict__ core) {
  const i64 b = blockIdx.x;
  if (b >= g) return;
  const int32_t j = col_sid[b];
  for (i64 e = ptr[j] + threadIdx.x; e < ptr[j + 1]; e += blockDim.x) {
    const int32_t a = pos_of_sid[row[e]];
    if (a >= 0) core[static_cast<i64>(a) * g + b] = val[e];
  }
}

using clk = std::chrono::steady_clock;

bool trace_on() { return trace_enabled(); }
// per-rank timings of the sharded part only (scripts/shard_model.py): one
// synchronisation per rank and phase, unlike the full trace
bool shard_timing() {
  static const bool on = std::getenv("PMMF_B200_SHARD_TIMING") != nullptr;
  return on || trace_enabled();
}
size_t mem_used_mb() {
  size_t f = 0, t = 0;
  cudaMemGetInfo(&f, &t);
  return (t - f) >> 20;
}
#define PMMF_TRACE(...)                 \
  do {                                  \
    if (trace_on()) {                   \
      std::fprintf(stderr, __VA_ARGS__); \
      std::fflush(stderr);              \
    }                                   \
  } while (0)
double ms_since(clk::time_point t) { return std::chrono::duration<double, std::milli>(clk::now() - t).count(); }

void validate(const pmmf_b200_params& p) {  // factorizer.hpp:44-50, clustering.hpp:36-40
  if (p.k < 2 || p.k > 8) fail(PMMF_INVALID_ARGUMENT, "FactorizeParams: k must be in [2, 8]");
  if (p.n_stages < 1) fail(PMMF_INVALID_ARGUMENT, "FactorizeParams: n_stages < 1");
  if (!(p.eta > 0.0 && p.eta < 1.0)) fail(PMMF_INVALID_ARGUMENT, "FactorizeParams: eta not in (0,1)");
  if (p.core_min < 1) fail(PMMF_INVALID_ARGUMENT, "FactorizeParams: core_min < 1");
  if (p.m_target < 1) fail(PMMF_INVALID_ARGUMENT, "ClusterParams: m_target < 1");
  if (p.c_min > p.c_max) fail(PMMF_INVALID_ARGUMENT, "ClusterParams: c_min > c_max");
  if (p.d_max < 0) fail(PMMF_INVALID_ARGUMENT, "ClusterParams: d_max < 0");
}

struct StreamGuard {
  cudaStream_t s = nullptr;
  StreamGuard() { PMMF_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~StreamGuard() {
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
};

// out[i] = b[a[i]] (relabel maps between two stage numberings: stage id ->
// global -> stage id)
__global__ void k_compose(i64 N, const int32_t* __restrict__ a, const int32_t* __restrict__ b,
                          int32_t* __restrict__ out) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < N) out[i] = b[a[i]];
}

}  // namespace


std::unique_ptr<Result> factorize_device(const pmmf_b200_coo* in, const pmmf_b200_params& p,
                                         const Comm* comm) {
  const Comm one;
  const Comm& C = comm ? *comm : one;
  if (comm && comm->device != in->device)
    fail(PMMF_INVALID_ARGUMENT, "factorize_sharded: input device differs from the communicator's");
  const int W = C.world();
  const std::vector<int> my_ranks = C.local_ranks();
  PMMF_CUDA(cudaSetDevice(in->device));
  const auto fn_start = clk::now();
  const uint64_t fresh0 = fresh_big_bytes().load();
  uint64_t reserved0 = 0;
  if (trace_on())
    (void)cudaMemPoolGetAttribute(lib_pool(in->device), cudaMemPoolAttrReservedMemCurrent, &reserved0);
  StreamGuard sg;
  cudaStream_t s = sg.s;
  const i64 n = in->n;
  if (n >= (i64{1} << 31) - 1) fail(PMMF_INVALID_ARGUMENT, "factorize: dimension exceeds 2^31 - 1");
  auto R = std::make_unique<Result>();
  R->n = n;
  R->k = p.k;
  R->params = p;

  // ---- input partition and from_triplets
  Numbering cur;
  {
    std::vector<std::vector<i64>> init;
    if (in->n_clusters == 0) {
      init.emplace_back(static_cast<size_t>(std::max<i64>(n, 0)));
      std::iota(init[0].begin(), init[0].end(), i64{0});
    } else {
      for (i64 u = 0; u < in->n_clusters; ++u)
        init.emplace_back(in->cluster_members + in->cluster_offsets[u], in->cluster_members + in->cluster_offsets[u + 1]);
    }
    cur.build(init, std::max<i64>(n, 0), s);
  }
  auto plap = [&, tp = clk::now()](const char* what) mutable {  // trace-mode prologue laps
    if (!trace_on()) return;
    PMMF_CUDA(cudaStreamSynchronize(s));
    PMMF_TRACE("[pmmf]   prologue.%s %.2f ms\n", what, ms_since(tp));
    tp = clk::now();
  };
  plap("numbering");
  Csc A;
  {
    const int64_t* rows = in->rows;
    const int64_t* cols = in->cols;
    const double* vals = in->vals;
    DBuf<int64_t> drow, dcol;
    DBuf<double> dval;
    if (!in->on_device && in->nnz > 0) {
      drow.alloc(in->nnz, s);
      dcol.alloc(in->nnz, s);
      dval.alloc(in->nnz, s);
      drow.upload(in->rows, in->nnz);
      dcol.upload(in->cols, in->nnz);
      dval.upload(in->vals, in->nnz);
      rows = drow.get();
      cols = dcol.get();
      vals = dval.get();
    }
    plap("upload");
    csc_from_coo(A, cur, std::max<i64>(n, 0), in->nnz, rows, cols, vals, s);
    plap("from_triplets");
  }
  validate(p);
  if (n < 1) fail(PMMF_INVALID_ARGUMENT, "factorize: empty matrix");
  {
    double asym = 0.0, fro = 0.0;
    csc_symmetry(A, cur, &asym, &fro, s);
    plap("symmetry");
    if (asym > 1e-9 * std::max(std::sqrt(fro), 1e-300))
      fail(PMMF_INVALID_ARGUMENT, "factorize: input matrix is not symmetric");
  }

  // ---- owned-column slabs (shard.cuh).  One GPU: one slab, the matrix.
  // Sharded: rank r keeps the columns it owns (full row range); the stage's
  // clustering, Gram, search and rotation passes run on them, and the
  // reblock moves columns to their new owners (all-to-all).  Before the
  // first stage: W contiguous column ranges of about equal nnz.
  const bool sharded = W > 1 || C.multi_process();
  std::vector<Csc> slab(my_ranks.size());
  std::vector<std::pair<i64, i64>> own(my_ranks.size());
  if (!sharded) {
    own[0] = {0, A.N};
    slab[0] = std::move(A);
  } else {
    const std::vector<i64> hp = A.ptr.to_host(A.N + 1);
    std::vector<i64> cut(static_cast<size_t>(W) + 1, A.N);
    cut[0] = 0;
    for (int r = 1; r < W; ++r) {
      const i64 target = A.nnz * r / W;
      cut[r] = std::max(cut[r - 1], static_cast<i64>(std::lower_bound(hp.begin(), hp.end(), target) - hp.begin()));
      cut[r] = std::min(cut[r], A.N);
    }
    for (size_t li = 0; li < my_ranks.size(); ++li) {
      own[li] = {cut[my_ranks[li]], cut[my_ranks[li] + 1]};
      slab_of(slab[li], A, own[li].first, own[li].second, s);
    }
    A = Csc();
  }
  auto slab_nnz = [&] {
    i64 t = 0;
    for (const Csc& x : slab) t += x.nnz;
    return t;
  };

  const auto run_start = clk::now();
  PMMF_TRACE("[pmmf] prologue (input numbering, from_triplets, symmetry) %.2f ms\n", ms_since(fn_start));
  std::vector<i64> active;
  for (i64 g = 0; g < n; ++g)
    if (cur.g2s[g] >= 0) active.push_back(g);
  R->hist.push_back(static_cast<i64>(active.size()));
  DBuf<uint8_t> d_active(n, s);
  DBuf<int32_t> d_rank(n, s);
  {
    std::vector<uint8_t> h(static_cast<size_t>(n), 0);
    for (i64 g : active) h[g] = 1;
    d_active.upload(h);
    d_rank.fill_bytes(0xff);
  }
  R->trivial = static_cast<i64>(active.size()) <= p.core_min;

  // one side stream for the rotation-record copies of every stage, one
  // retired-id scratch mask (both were per stage: ~1 ms of fixed host cost each)
  struct SideStream {
    cudaStream_t st = nullptr;
    ~SideStream() {
      if (st) cudaStreamDestroy(st);
    }
  } side_holder;
  PMMF_CUDA(cudaStreamCreateWithFlags(&side_holder.st, cudaStreamNonBlocking));
  const cudaStream_t side = side_holder.st;
  std::vector<uint8_t> gone(static_cast<size_t>(std::max<i64>(n, 1)), 0);
  // reserved once: reserve(size + ne) per stage reallocated and copied the
  // whole list every stage (2-5 ms each, also in the tiny late stages)
  R->diag.reserve(static_cast<size_t>(std::max<i64>(n, 0)));
  for (int stage_no = 1; stage_no <= p.n_stages && !R->trivial; ++stage_no) {
    if (static_cast<i64>(active.size()) <= p.core_min) break;
    const auto t_stage = clk::now();
    double ph0[5];
    std::copy(R->phases, R->phases + 5, ph0);
    // ---- clustering on the pre-reblock matrix
    auto t0 = clk::now();
    const uint64_t cpath[2] = {0xC1u, static_cast<uint64_t>(stage_no)};
    SlabSet ss;
    for (const Csc& x : slab) ss.slabs.push_back(&x);
    ss.own = own;
    ss.comm = sharded ? &C : nullptr;
    ClusterOut co = cluster_columns_dev(ss, cur, active, n, p.m_target, p.c_min, p.c_max, p.d_max,
                                        p.bypass_enabled != 0, derive(p.seed, cpath), s);
    R->phases[0] += ms_since(t0);
    const i64 rc = static_cast<i64>(co.sizes.size());
    std::vector<i64> stage_off(1, 0);
    for (i64 c : co.sizes) stage_off.push_back(stage_off.back() + c);
    if (!co.bypassed.empty()) stage_off.push_back(stage_off.back() + static_cast<i64>(co.bypassed.size()));

    // ---- reblock to the stage numbering (relabel maps composed on the device)
    t0 = clk::now();
    Numbering nxt;
    nxt.build_device(std::move(co.members), std::move(stage_off), n, s);
    {
      DBuf<int32_t> dmap(std::max<i64>(cur.size(), 1), s), dn2o(std::max<i64>(nxt.size(), 1), s);
      PMMF_LAUNCH(k_compose, blocks_for(cur.size(), kThreads), kThreads, 0, s, cur.size(), cur.d_s2g.get(),
                  nxt.d_g2s.get(), dmap.get());
      PMMF_LAUNCH(k_compose, blocks_for(nxt.size(), kThreads), kThreads, 0, s, nxt.size(), nxt.d_s2g.get(),
                  cur.d_g2s.get(), dn2o.get());
      for (size_t li = 0; li < slab.size(); ++li) {  // each slab relabelled in place (its columns stay)
        const auto t_r = clk::now();
        Csc B;
        reblock(B, slab[li], dmap, dn2o, nxt.size(), s);
        slab[li] = std::move(B);
        if (sharded && shard_timing()) {
          PMMF_CUDA(cudaStreamSynchronize(s));
          std::fprintf(stderr, "[pmmf] shard stage %d rank %d: reblock %.3f ms\n", stage_no + 1, my_ranks[li],
                       ms_since(t_r));
        }
      }
    }
    cur = std::move(nxt);
    PMMF_CUDA(cudaStreamSynchronize(s));
    R->phases[4] += ms_since(t0);
    PMMF_TRACE("[pmmf] stage %d: reblock %.2f ms (%lld entries)\n", stage_no + 1, ms_since(t0),
               static_cast<long long>(slab_nnz()));

    Result::Stage st;
    st.off = cur.off;
    st.members = cur.s2g;
    st.bypassed = co.bypassed;

    // ---- budgets (factorizer.hpp:463-479)
    std::vector<i64> budget(static_cast<size_t>(rc), 0);
    i64 planned = 0;
    for (i64 u = 0; u < rc; ++u) {
      const i64 c = cur.off[u + 1] - cur.off[u];
      i64 b = c < p.k ? 0 : static_cast<i64>(std::floor(p.eta * static_cast<double>(c)));
      b = std::min(b, std::max<i64>(0, c - (p.k - 1)));
      budget[u] = b;
      planned += b;
    }
    const i64 allowance = std::max<i64>(0, static_cast<i64>(active.size()) - p.core_min);
    while (planned > allowance) {
      i64 arg = 0;
      for (i64 u = 1; u < rc; ++u)
        if (budget[u] > budget[arg]) arg = u;
      --budget[arg];
      --planned;
    }
    std::vector<int64_t> out_base(static_cast<size_t>(rc) + 1, 0);
    for (i64 u = 0; u < rc; ++u) out_base[u + 1] = out_base[u] + budget[u];
    const i64 slots = out_base[rc];
    // ---- cluster ownership (shard.cuh): rank r owns clusters [lo[r], lo[r+1])
    const i64 nclu = cur.clusters();
    std::vector<i64> lo{0, nclu};
    if (W > 1) {
      std::vector<i64> csz(static_cast<size_t>(nclu)), cnz(static_cast<size_t>(nclu), 0);
      for (const Csc& x : slab) {  // this rank's entries per new cluster, summed over ranks
        const std::vector<i64> e = cluster_ptr(x, cur.off, s);
        for (i64 u = 0; u < nclu; ++u) cnz[u] += e[u + 1] - e[u];
      }
      if (C.multi_process()) {
        DBuf<int64_t> d(nclu, s);
        d.upload(cnz);
        allreduce_sum_i64(d.get(), nclu, C, s);
        cnz = d.to_host(nclu);
      }
      for (i64 u = 0; u < nclu; ++u) csz[u] = cur.off[u + 1] - cur.off[u];
      lo = shard_ranges(csz, cnz, W);
    }
    if (sharded) {
      // the all-to-all of the reblock: columns to the owners of their clusters
      const auto t_x = clk::now();
      std::vector<i64> dest(static_cast<size_t>(W) + 1);
      for (int r = 0; r <= W; ++r) dest[r] = cur.off[std::min(lo[r], nclu)];
      if (shard_timing() && C.virt) {  // ingress per rank of the all-to-all (scripts/shard_model.py)
        std::vector<i64> in_bytes(static_cast<size_t>(W), 0);
        DBuf<i64> idx(W + 1, s), v(W + 1, s);
        idx.upload(dest);
        for (size_t si = 0; si < slab.size(); ++si) {
          const std::vector<i64> at = cluster_ptr(slab[si], dest, s);
          for (int d = 0; d < W; ++d)
            if (d != my_ranks[si]) in_bytes[d] += 12 * (at[d + 1] - at[d]) + 4 * (dest[d + 1] - dest[d]);
        }
        std::fprintf(stderr, "[pmmf] shard stage %d: all-to-all ingress max %lld bytes\n", stage_no,
                     static_cast<long long>(*std::max_element(in_bytes.begin(), in_bytes.end())));
        PMMF_CUDA(cudaStreamSynchronize(s));
      }
      const auto t_rd = clk::now();
      redistribute(slab, dest, cur.size(), C, s);
      if (shard_timing()) {
        PMMF_CUDA(cudaStreamSynchronize(s));
        std::fprintf(stderr, "[pmmf] shard stage %d: exchange %.3f ms\n", stage_no, ms_since(t_rd));
      }
      for (size_t li = 0; li < my_ranks.size(); ++li) own[li] = {dest[my_ranks[li]], dest[my_ranks[li] + 1]};
      PMMF_CUDA(cudaStreamSynchronize(s));
      R->phases[4] += ms_since(t_x);
    }
    auto seg_of = [&](auto&& f) {  // per-rank segment bounds from a cluster-indexed prefix f(u)
      std::vector<i64> g(static_cast<size_t>(W) + 1);
      for (int r = 0; r <= W; ++r) g[r] = f(std::min(lo[r], rc));
      return g;
    };

    // ---- Gram + search, in batches of clusters whose tiles fit in memory
    SearchOut so;
    so.nrot.alloc(std::max<i64>(rc, 1), s);
    so.nelim.alloc(std::max<i64>(rc, 1), s);
    so.nrot.zero();
    so.nelim.zero();
    so.rot_loc.alloc(std::max<i64>(slots * p.k, 1), s);
    so.rot_q.alloc(std::max<i64>(slots * p.k * p.k, 1), s);
    so.rot_level.alloc(std::max<i64>(slots, 1), s);
    so.elim_loc.alloc(std::max<i64>(slots, 1), s);
    so.error.alloc(1, s);
    so.error.zero();
    DBuf<int64_t> d_out_base(rc + 1, s), d_coff(rc + 1, s);
    d_out_base.upload(out_base);
    d_coff.upload(cur.off.data(), rc + 1);
    {
      const i64 budget_elems =
          std::max<i64>(i64{1} << 20, static_cast<i64>(static_cast<double>(available_bytes()) * 0.55) / 16);
      double gram_ms = 0.0, search_ms = 0.0;
      for (size_t li = 0; li < my_ranks.size(); ++li) {
      const int me = my_ranks[li];
      const auto t_rank = clk::now();
      const double gs0 = gram_ms + search_ms;
      const i64 u_end = std::min(lo[me + 1], rc);
      i64 u0 = std::min(lo[me], rc);
      while (u0 < u_end) {
        i64 u1 = u0, elems = 0, max_c = 0;
        std::vector<i64> tile_off(1, 0);
        while (u1 < u_end) {
          const i64 c = cur.off[u1 + 1] - cur.off[u1];
          if (u1 > u0 && elems + c * c > budget_elems) break;
          elems += c * c;
          max_c = std::max(max_c, c);
          tile_off.push_back(elems);
          ++u1;
        }
        auto tg = clk::now();
        DBuf<double> G(std::max<i64>(elems, 1), s), D(std::max<i64>(elems, 1), s);
        G.zero();
        D.zero();
        // gram_tiles wants tile_off indexed by absolute u
        std::vector<i64> toff(static_cast<size_t>(u1) + 1, 0);
        for (i64 u = u0; u <= u1; ++u) toff[u] = tile_off[u - u0];
        gram_tiles(slab[li], cur.off, u0, u1, toff, G.get(), D.get(), s);
        PMMF_CUDA(cudaStreamSynchronize(s));
        gram_ms += ms_since(tg);
        auto ts = clk::now();
        const i64 nb = u1 - u0;
        SearchBatch sb;
        std::vector<int64_t> hc(nb), ht(nb), hb(nb), hob(nb);
        std::vector<uint64_t> hs(nb);
        for (i64 u = u0; u < u1; ++u) {
          hc[u - u0] = cur.off[u + 1] - cur.off[u];
          ht[u - u0] = tile_off[u - u0];
          hb[u - u0] = budget[u];
          hob[u - u0] = out_base[u];
          const uint64_t spath[3] = {0xF0u, static_cast<uint64_t>(stage_no), static_cast<uint64_t>(u)};
          hs[u - u0] = derive(p.seed, spath);
        }
        sb.c.alloc(nb, s);
        sb.tile.alloc(nb, s);
        sb.budget.alloc(nb, s);
        sb.seed.alloc(nb, s);
        sb.out_base.alloc(nb, s);
        sb.c.upload(hc);
        sb.h_c = hc;
        sb.tile.upload(ht);
        sb.budget.upload(hb);
        sb.seed.upload(hs);
        sb.out_base.upload(hob);
        {
          // largest clusters first: the search is quadratic in c and the
          // kernel ends with its slowest CTA
          std::vector<int32_t> ord(static_cast<size_t>(nb));
          std::iota(ord.begin(), ord.end(), 0);
          std::stable_sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) { return hc[x] > hc[y]; });
          sb.order.alloc(nb, s);
          sb.order.upload(ord);
        }
        search_clusters(sb, u0, nb, p.k, p.eta, G.get(), D.get(), std::max<i64>(max_c, 1), so, s);
        PMMF_CUDA(cudaStreamSynchronize(s));
        search_ms += ms_since(ts);
        u0 = u1;
      }
      if (W > 1 && shard_timing())  // per-rank cost of the sharded part (scripts/shard_model.py)
        std::fprintf(stderr, "[pmmf] shard stage %d rank %d: gram+search %.3f ms (%.3f wall) clusters [%lld,%lld)\n", stage_no,
                   me, gram_ms + search_ms - gs0, ms_since(t_rank), static_cast<long long>(lo[me]),
                   static_cast<long long>(lo[me + 1]));
      }
      R->phases[1] += gram_ms;
      R->phases[2] += search_ms;
      PMMF_TRACE("[pmmf] stage %d: gram %.2f ms, search %.2f ms\n", stage_no, gram_ms, search_ms);
    }
    if (C.multi_process()) {
      // exchange 1: every rank's clusters' rotation slots and counts
      const auto t_x = clk::now();
      const auto cseg = seg_of([](i64 u) { return u; });
      const auto sseg = seg_of([&](i64 u) { return out_base[u]; });
      bcast_segments(so.nrot.get(), sizeof(int32_t), cseg, C, s);
      bcast_segments(so.nelim.get(), sizeof(int32_t), cseg, C, s);
      bcast_segments(so.rot_loc.get(), sizeof(int32_t) * p.k, sseg, C, s);
      bcast_segments(so.rot_q.get(), sizeof(double) * p.k * p.k, sseg, C, s);
      bcast_segments(so.rot_level.get(), sizeof(int32_t), sseg, C, s);
      bcast_segments(so.elim_loc.get(), sizeof(int32_t), sseg, C, s);
      allreduce_max_i32(so.error.get(), C, s);
      PMMF_CUDA(cudaStreamSynchronize(s));
      R->phases[2] += ms_since(t_x);
    }
    const auto t_asm = clk::now();
    if (so.error.to_host(1)[0]) fail(PMMF_INVALID_ARGUMENT, "rotation_from_gram: input not symmetric");
    std::vector<int32_t> nrot = so.nrot.to_host(std::max<i64>(rc, 1));
    std::vector<int32_t> nelim = so.nelim.to_host(std::max<i64>(rc, 1));
    std::vector<int32_t> elim_loc = so.elim_loc.to_host(std::max<i64>(slots, 1));
    std::vector<int32_t> order_sid;  // eliminated stage ids, stage elimination order
    std::vector<int32_t> order_g;
    {
      size_t total = 0;
      for (i64 u = 0; u < rc; ++u) total += static_cast<size_t>(nelim[u]);
      order_sid.resize(total);
      order_g.resize(total);
      size_t w = 0;
      for (i64 u = 0; u < rc; ++u) {
        const i64 o = cur.off[u];
        const int32_t* el = elim_loc.data() + out_base[u];
        for (i64 e = 0; e < nelim[u]; ++e, ++w) {
          const i64 sid = o + el[e];
          order_sid[w] = static_cast<int32_t>(sid);
          order_g[w] = static_cast<int32_t>(cur.s2g[sid]);
        }
      }
    }
    // The rotation records (global ids, k x k blocks) are only reported:
    // a worker thread copies them through pinned staging on a side stream and
    // assembles them while the device runs the stage apply (which reads the
    // same device arrays, never writes them).
    std::future<void> records;
    {
      int dev = 0;
      PMMF_CUDA(cudaGetDevice(&dev));
      cudaEvent_t ready = nullptr;
      PMMF_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
      PMMF_CUDA(cudaEventRecord(ready, s));
      const int32_t* d_loc = so.rot_loc.get();
      const double* d_q = so.rot_q.get();
      const int k = p.k;
      records = std::async(std::launch::async, [&st, &nrot, &out_base, &cur, rc, slots, k, d_loc, d_q, ready, dev, side]() {
        PMMF_CUDA(cudaSetDevice(dev));
        PMMF_CUDA(cudaStreamWaitEvent(side, ready, 0));
        const size_t nl = static_cast<size_t>(std::max<i64>(slots * k, 1));
        const size_t nq = static_cast<size_t>(std::max<i64>(slots * k * k, 1));
        PinnedSlot& pl = PinnedSlot::get(0);
        PinnedSlot& pq = PinnedSlot::get(1);
        std::lock_guard<std::mutex> gl(pl.mu), gq(pq.mu);
        auto* hl = static_cast<int32_t*>(pl.reserve(nl * sizeof(int32_t)));
        auto* hq = static_cast<double*>(pq.reserve(nq * sizeof(double)));
        std::vector<int32_t> vl;
        std::vector<double> vq;
        if (!hl || !hq) {  // no pinned memory: pageable copies
          vl.resize(nl);
          vq.resize(nq);
          hl = vl.data();
          hq = vq.data();
        }
        PMMF_CUDA(cudaMemcpyAsync(hl, d_loc, nl * sizeof(int32_t), cudaMemcpyDeviceToHost, side));
        PMMF_CUDA(cudaMemcpyAsync(hq, d_q, nq * sizeof(double), cudaMemcpyDeviceToHost, side));
        PMMF_CUDA(cudaStreamSynchronize(side));
        cudaEventDestroy(ready);
        i64 total = 0;
        for (i64 u = 0; u < rc; ++u) total += nrot[u];
        st.rot_idx.resize(static_cast<size_t>(total * k));
        st.rot_q.resize(static_cast<size_t>(total * k * k));
        i64 w = 0;
        for (i64 u = 0; u < rc; ++u)
          for (i64 t = 0; t < nrot[u]; ++t, ++w) {
            const i64 sl = out_base[u] + t;
            for (int a = 0; a < k; ++a) st.rot_idx[w * k + a] = cur.s2g[cur.off[u] + hl[sl * k + a]];
            std::copy(hq + sl * k * k, hq + (sl + 1) * k * k, st.rot_q.begin() + w * k * k);
          }
      });
    }

    PMMF_TRACE("[pmmf] stage %d: host assembly of the rotation records %.2f ms\n", stage_no, ms_since(t_asm));
    // ---- stage apply: column side, transpose, row side, transpose
    t0 = clk::now();
    const i64 ne = static_cast<i64>(order_g.size());
    DBuf<int32_t> dsid(std::max<i64>(ne, 1), s), dg(std::max<i64>(ne, 1), s);
    dsid.upload(order_sid);
    dg.upload(order_g);
    DBuf<double> mass(std::max<i64>(ne, 1), s), diag(std::max<i64>(ne, 1), s);
    bool residual_done = false;
    {
      LevelPlan plan;
      build_plan(plan, so, d_out_base, d_coff, rc, slots, p.k, s);
      if (plan.max_level > 0) {
        const i64 N = cur.size();
        std::vector<i64> slot_base(static_cast<size_t>(cur.clusters()) + 1, slots);
        for (i64 u = 0; u <= rc; ++u) slot_base[u] = out_base[u];
        const i64 avail = available_bytes();
        i64 chunk = std::max<i64>(i64{1} << 22, avail / 10 / 32);
        if (const char* e = std::getenv("PMMF_B200_CHUNK_NNZ")) chunk = std::atoll(e);  // test hook
        // trace-mode sub-phase timer (synchronises only when tracing)
        auto tl = clk::now();
        auto lap = [&](const char* what) {
          if (!trace_on()) return;
          PMMF_CUDA(cudaStreamSynchronize(s));
          PMMF_TRACE("[pmmf]   apply.%s %.2f ms\n", what, ms_since(tl));
          tl = clk::now();
        };
        lap("plan");
        // Retired ids: their rotated rows/columns feed only the residual.
        DBuf<uint8_t> keep_row(N, s);
        {
          std::vector<uint8_t> kr(static_cast<size_t>(N), 1);
          for (int32_t sid : order_sid) kr[sid] = 0;
          keep_row.upload(kr);
        }
        // Row pass with the residual masses taken from its final columns
        // (rows of A'), which then keep only the surviving rows.
        MassSpec ms;
        DBuf<int32_t> row_rank(N, s), col_key(N, s);
        if (ne > 0) {
          row_rank.fill_bytes(0xff);
          col_key.fill_bytes(0x7f);
          PMMF_LAUNCH(k_mass_keys, blocks_for(ne, kThreads), kThreads, 0, s, ne, dsid.get(), row_rank.get(),
                      col_key.get());
          mass.zero();
          diag.zero();
          ms.row_rank = row_rank.get();
          ms.col_key = col_key.get();
          ms.mass = mass.get();
          ms.diag = diag.get();
          ms.chunk_nnz = chunk;
          ms.n_retired = ne;
        }
        // One column slab per rank (shard.cuh): the rank's clusters' columns
        // through the column pass, transpose, row pass (all rotations) and
        // transpose back.  With one rank the slab is the whole matrix.
        std::vector<Csc> slabs;
        for (size_t li = 0; li < my_ranks.size(); ++li) {
          const int me = my_ranks[li];
          if (W > 1 && shard_timing()) PMMF_CUDA(cudaStreamSynchronize(s));
          const auto t_rank = clk::now();
          std::vector<Piece> pieces;
          const i64 nnz_in = std::max<i64>(slab[li].nnz, 1);
          rotate_pass(pieces, slab[li], cur.off, slot_base, plan, nullptr, nullptr, i64{1} << 62, 24.0, nullptr, s, lo[me],
                      lo[me + 1]);
          lap("column_pass");
          slab[li] = Csc();
          Csc T;
          transpose_pieces(T, pieces, N, nullptr, chunk, s);
          pieces.clear();
          lap("transpose_1");
          const i64 tn = T.nnz;
          // The row pass grows its columns about as much as the column pass
          // did (measured ratio); size its arena and batches from that.
          const double growth =
              1.4 * std::max(2.0, static_cast<double>(tn) / static_cast<double>(nnz_in));
          // (free memory re-read: T and the retired masks now hold their share)
          const i64 avail_row = available_bytes();
          double frac = 0.2;  // share of free memory for one batch's arena
          if (const char* e = std::getenv("PMMF_B200_ARENA_FRAC")) frac = std::atof(e);
          i64 batch = std::max<i64>(i64{1} << 24,
                                    static_cast<i64>(frac * static_cast<double>(avail_row) / (12.0 * growth)));
          if (const char* e = std::getenv("PMMF_B200_BATCH_NNZ")) batch = std::atoll(e);  // test hook
          PMMF_TRACE("[pmmf] stage %d rank %d: column pass -> %lld entries, batch=%lld mem=%zuMB\n", stage_no, me,
                     static_cast<long long>(tn), static_cast<long long>(batch), mem_used_mb());
          if (ne > 0) {  // this slab's retired rows: its own clusters' eliminations (cluster-major ranks)
            i64 e0 = 0, e1 = 0;
            for (i64 u = 0; u < std::min(lo[me + 1], rc); ++u) (u < lo[me] ? e0 : e1) += nelim[u];
            ms.rank_base = e0;
            ms.n_retired = e1;
          }
          rotate_pass(pieces, T, cur.off, slot_base, plan, keep_row.get(), nullptr, batch, growth,
                      ne > 0 && ms.n_retired > 0 ? &ms : nullptr, s);
          T = Csc();
          lap("row_pass");
          i64 stored = 0;
          for (const Piece& P : pieces) stored += P.nnz;
          PMMF_TRACE("[pmmf] stage %d rank %d: row pass stored %lld entries in %zu pieces, mem=%zuMB\n", stage_no,
                     me, static_cast<long long>(stored), pieces.size(), mem_used_mb());
          // The next stage reads only the surviving columns of A' (all rows).
          slabs.emplace_back();
          transpose_pieces(slabs.back(), pieces, N, nullptr, chunk, s);
          lap("transpose_2");
          if (W > 1 && shard_timing()) {
            PMMF_CUDA(cudaStreamSynchronize(s));
            std::fprintf(stderr, "[pmmf] shard stage %d rank %d: apply %.3f ms, slab %lld entries\n", stage_no, me,
                       ms_since(t_rank), static_cast<long long>(slabs.back().nnz));
          }
        }
        if (ne > 0) {  // retired ids leave the active set
          PMMF_LAUNCH(k_mark, blocks_for(ne, kThreads), kThreads, 0, s, ne, dg.get(), d_active.get(), d_rank.get(), 0);
          residual_done = true;
        }
        // the owned columns of A'' stay on their rank (the next reblock moves
        // them); across processes the owned eliminations' masses and
        // diagonals (cluster-major) are broadcast
        slab = std::move(slabs);
        if (ne > 0 && C.multi_process()) {
          std::vector<i64> epre(static_cast<size_t>(rc) + 1, 0);
          for (i64 u = 0; u < rc; ++u) epre[u + 1] = epre[u] + nelim[u];
          const auto eseg = seg_of([&](i64 u) { return epre[u]; });
          bcast_segments(mass.get(), sizeof(double), eseg, C, s);
          bcast_segments(diag.get(), sizeof(double), eseg, C, s);
        }
        PMMF_TRACE("[pmmf] stage %d: A' %lld entries, mem=%zuMB\n", stage_no, static_cast<long long>(slab_nnz()),
                   mem_used_mb());
      }
    }
    PMMF_CUDA(cudaStreamSynchronize(s));
    R->phases[3] += ms_since(t0);
    PMMF_TRACE("[pmmf] stage %d: apply %.2f ms\n", stage_no, ms_since(t0));
    const auto t_res = clk::now();

    // ---- residual accounting against the end-of-stage matrix
    if (ne > 0) {
      if (!residual_done) {
        PMMF_LAUNCH(k_mark, blocks_for(ne, kThreads), kThreads, 0, s, ne, dg.get(), d_active.get(), d_rank.get(), 1);
        for (size_t li = 0; li < slab.size(); ++li)
          PMMF_LAUNCH(k_residual, blocks_for(ne * 32, kThreads), kThreads, 0, s, ne, dsid.get(), slab[li].ptr.get(),
                      slab[li].row.get(), slab[li].val.get(), cur.d_s2g.get(), d_active.get(), d_rank.get(), mass.get(),
                      diag.get(), own[li].first, own[li].second);
        if (C.multi_process()) {  // zeros elsewhere: the sums are the owners' values
          allreduce_sum_f64(mass.get(), ne, C, s);
          allreduce_sum_f64(diag.get(), ne, C, s);
        }
        PMMF_LAUNCH(k_mark, blocks_for(ne, kThreads), kThreads, 0, s, ne, dg.get(), d_active.get(), d_rank.get(), 0);
      }
      PinnedSlot& ps = PinnedSlot::get(2);
      std::lock_guard<std::mutex> lk(ps.mu);
      auto* hmd = static_cast<double*>(ps.reserve(sizeof(double) * 2 * static_cast<size_t>(ne)));
      std::vector<double> fallback;
      if (!hmd) {
        fallback.resize(2 * static_cast<size_t>(ne));
        hmd = fallback.data();
      }
      PMMF_CUDA(cudaMemcpyAsync(hmd, mass.get(), sizeof(double) * ne, cudaMemcpyDeviceToHost, s));
      PMMF_CUDA(cudaMemcpyAsync(hmd + ne, diag.get(), sizeof(double) * ne, cudaMemcpyDeviceToHost, s));
      PMMF_CUDA(cudaStreamSynchronize(s));
      PMMF_TRACE("[pmmf]   bookkeeping: masses on the host at %.2f ms\n", ms_since(t_res));
      const double* hm = hmd;
      const double* hd = hmd + ne;
      st.elim_idx.assign(order_g.begin(), order_g.end());
      st.elim_diag.assign(hd, hd + ne);
      st.elim_mass.assign(hm, hm + ne);
      for (i64 r = 0; r < ne; ++r) {
        R->residual_sq += 2.0 * hm[r];
        R->diag.push_back({order_g[r], hd[r]});
      }
    }
    PMMF_TRACE("[pmmf]   bookkeeping: stage records filled at %.2f ms\n", ms_since(t_res));
    {
      for (int32_t g : order_g) gone[g] = 1;
      size_t w = 0;  // in place: no 4-8 MB allocation (and its page faults) per stage
      for (size_t i = 0; i < active.size(); ++i) {
        const i64 g = active[i];
        if (!gone[g]) active[w++] = g;
      }
      active.resize(w);
      for (int32_t g : order_g) gone[g] = 0;
    }
    PMMF_TRACE("[pmmf]   bookkeeping: active set filtered at %.2f ms\n", ms_since(t_res));
    records.get();  // rotation records assembled (rethrows a copy failure)
    PMMF_TRACE("[pmmf] stage %d: residual + bookkeeping %.2f ms\n", stage_no, ms_since(t_res));
    if (trace_on()) {
      double in_phases = 0.0;
      for (int i = 0; i < 5; ++i) in_phases += R->phases[i] - ph0[i];
      PMMF_TRACE("[pmmf] stage %d: wall %.2f ms, outside the five phases %.2f ms\n", stage_no, ms_since(t_stage),
                 ms_since(t_stage) - in_phases);
    }
    R->hist.push_back(static_cast<i64>(active.size()));
    R->info.push_back({stage_no, rc, static_cast<i64>(st.bypassed.size()),
                       static_cast<i64>(st.rot_idx.size()) / p.k, ne, static_cast<i64>(active.size()),
                       static_cast<i64>(co.max_depth)});
    R->stages.push_back(std::move(st));
  }

  if (static_cast<i64>(active.size()) > p.core_cap)
    fail(PMMF_NUMERIC, "factorize: core of size " + std::to_string(active.size()) + " exceeds the cap of " +
                           std::to_string(p.core_cap) + "; raise core_cap or add stages");
  const i64 g = static_cast<i64>(active.size());
  R->core_idx = active;
  R->core.assign(static_cast<size_t>(g * g), 0.0);
  if (g > 0) {
    std::vector<int32_t> col_sid(static_cast<size_t>(g)), pos(static_cast<size_t>(cur.size()), -1);
    const std::vector<i64>& g2s_h = cur.host_g2s();
    for (i64 a = 0; a < g; ++a) {
      col_sid[a] = static_cast<int32_t>(g2s_h[active[a]]);
      pos[col_sid[a]] = static_cast<int32_t>(a);
    }
    DBuf<int32_t> dcs(g, s), dpos(std::max<i64>(cur.size(), 1), s);
    dcs.upload(col_sid);
    dpos.upload(pos);
    DBuf<double> dcore(g * g, s);
    dcore.zero();
    for (const Csc& x : slab)  // other ranks' columns are empty in a slab
      PMMF_LAUNCH(k_core, static_cast<unsigned>(g), 128, 0, s, g, dcs.get(), x.ptr.get(), x.row.get(), x.val.get(),
                  dpos.get(), dcore.get());
    allreduce_sum_f64(dcore.get(), g * g, C, s);
    R->core = dcore.to_host(g * g);
  }
  {
    // order by global index (each retired index appears once): a counting
    // placement instead of an O(n log n) sort of ~10^6 pairs
    std::vector<double> dv(static_cast<size_t>(n), 0.0);
    std::vector<uint8_t> has(static_cast<size_t>(n), 0);
    for (const auto& [idx, v] : R->diag) {
      dv[idx] = v;
      has[idx] = 1;
    }
    size_t w = 0;
    for (i64 idx = 0; idx < n; ++idx)
      if (has[idx]) R->diag[w++] = {idx, dv[idx]};
    if (w != R->diag.size()) fail(PMMF_INTERNAL, "factorize: an index was retired twice");
  }
  PMMF_CUDA(cudaStreamSynchronize(s));
  R->phases[5] = ms_since(run_start);
  PMMF_TRACE("[pmmf] factorize total %.2f ms (stage loop + core %.2f ms)\n", ms_since(fn_start), R->phases[5]);
  if (trace_on()) {
    uint64_t reserved1 = 0;
    (void)cudaMemPoolGetAttribute(lib_pool(in->device), cudaMemPoolAttrReservedMemCurrent, &reserved1);
    PMMF_TRACE("[pmmf] memory: %llu MB of large blocks missed the cache, pool reserved %+lld MB\n",
               static_cast<unsigned long long>((fresh_big_bytes().load() - fresh0) >> 20),
               static_cast<long long>((static_cast<int64_t>(reserved1) - static_cast<int64_t>(reserved0)) >> 20));
  }
  return R;
}

}  // namespace pmmf_b200
