// gram.cu — per-cluster Gram matrices G_u = A[:,B_u]^T A[:,B_u]
// (blocked_matrix.hpp:238-254) and diagonal blocks D_u = A[B_u,B_u]
// (:257-266) as dense column-major c_u x c_u tiles.
//
// Bitwise order: G[a][b] is the sequential sum over
// the rows of the stage numbering of A[r][a]*A[r][b].  The cluster's column
// block is re-sorted by (row, column) once (segmented radix sort carrying
// the CSC entry index), every CSC entry learns the row-run that holds its
// row, and then a warp owns output column a: it walks column a's entries in
// row order and, per entry, adds the products with its row-run into
// G[:,a] — lanes on distinct b, rows strictly in order.  Work is
// sum_r deg_u(r)^2, the reference's own product count.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>

#include "engine.cuh"

namespace pmmf_b200 {

namespace {

constexpr int kThreads = 256;

// Keys (row << 32 | local col) and payload (entry index) for the entries of
// clusters [u0,u1).
__global__ void k_gram_keys(i64 e0, i64 ne, const i64* __restrict__ ptr, i64 col0, i64 ncols,
                            const int32_t* __restrict__ row, const int32_t* __restrict__ col_cluster_off,
                            uint64_t* __restrict__ keys, uint32_t* __restrict__ idx) {
  // one warp per column
  const i64 w = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= ncols) return;
  const i64 J = col0 + w;
  const uint64_t local = static_cast<uint64_t>(J - col_cluster_off[w]);
  for (i64 e = ptr[J] + lane; e < ptr[J + 1]; e += 32) {
    keys[e - e0] = (static_cast<uint64_t>(row[e]) << 32) | local;
    idx[e - e0] = static_cast<uint32_t>(e - e0);
  }
}

// Row runs of the sorted segment: the head of each run stamps [lo,hi) on
// every member, indexed by the member's original CSC entry.
__global__ void k_runs(i64 ne, const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx,
                       const int64_t* __restrict__ seg_of, const int64_t* __restrict__ seg_begin,
                       const int64_t* __restrict__ seg_end, const double* __restrict__ val_base,
                       int32_t* __restrict__ run_lo, int32_t* __restrict__ run_hi, int32_t* __restrict__ csr_col,
                       double* __restrict__ csr_val) {
  const i64 p = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (p >= ne) return;
  csr_col[p] = static_cast<int32_t>(keys[p] & 0xffffffffu);
  csr_val[p] = val_base[idx[p]];
  const i64 sb = seg_begin[seg_of[p]];
  const uint32_t r = static_cast<uint32_t>(keys[p] >> 32);
  if (p > sb && static_cast<uint32_t>(keys[p - 1] >> 32) == r) return;
  const i64 se = seg_end[seg_of[p]];
  i64 q = p + 1;
  while (q < se && static_cast<uint32_t>(keys[q] >> 32) == r) ++q;
  for (i64 t = p; t < q; ++t) {
    run_lo[idx[t]] = static_cast<int32_t>(p);
    run_hi[idx[t]] = static_cast<int32_t>(q);
  }
}

__global__ void k_seg_of(i64 ne, const int64_t* __restrict__ seg_begin, i64 nseg, int64_t* __restrict__ seg_of) {
  const i64 p = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (p >= ne) return;
  i64 lo = 0, hi = nseg;  // last seg with begin <= p
  while (hi - lo > 1) {
    const i64 mid = (lo + hi) >> 1;
    if (seg_begin[mid] <= p) lo = mid; else hi = mid;
  }
  seg_of[p] = lo;
}

__global__ void k_gather_ptr(i64 n, const int64_t* __restrict__ cols, const i64* __restrict__ ptr, i64 e0,
                             int64_t* __restrict__ out) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = ptr[cols[i]] - e0;
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
  const i64 a = J - col_cluster_off[w];
  const i64 c = col_c[w];
  double* Gcol = G + col_tile[w] + a * c;
  for (i64 e = ptr[J]; e < ptr[J + 1]; ++e) {
    const double va = val[e];
    const int32_t lo = run_lo[e - e0], hi = run_hi[e - e0];
    for (int32_t q = lo + lane; q < hi; q += 32) {
      const int32_t b = csr_col[q];
      Gcol[b] = dadd(Gcol[b], dmul(va, csr_val[q]));
    }
    __syncwarp();
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

}  // namespace

void gram_tiles(const Csc& a, const std::vector<i64>& off, i64 u0, i64 u1, const std::vector<i64>& tile_off,
                double* G, double* D, cudaStream_t s) {
  const i64 col0 = off[u0], ncols = off[u1] - off[u0];
  if (ncols <= 0) return;
  std::vector<i64> hptr(2);
  PMMF_CUDA(cudaMemcpyAsync(&hptr[0], a.ptr.get() + col0, sizeof(i64), cudaMemcpyDeviceToHost, s));
  PMMF_CUDA(cudaMemcpyAsync(&hptr[1], a.ptr.get() + col0 + ncols, sizeof(i64), cudaMemcpyDeviceToHost, s));
  // per-column cluster info
  std::vector<int32_t> cco(static_cast<size_t>(ncols)), cc(static_cast<size_t>(ncols));
  std::vector<int64_t> ct(static_cast<size_t>(ncols));
  for (i64 u = u0; u < u1; ++u)
    for (i64 J = off[u]; J < off[u + 1]; ++J) {
      cco[J - col0] = static_cast<int32_t>(off[u]);
      cc[J - col0] = static_cast<int32_t>(off[u + 1] - off[u]);
      ct[J - col0] = tile_off[u] - tile_off[u0];
    }
  DBuf<int32_t> dcco(ncols, s), dcc(ncols, s);
  DBuf<int64_t> dct(ncols, s);
  dcco.upload(cco);
  dcc.upload(cc);
  dct.upload(ct);
  PMMF_CUDA(cudaStreamSynchronize(s));
  const i64 e0 = hptr[0], ne = hptr[1] - hptr[0];
  PMMF_LAUNCH(k_diag_block, blocks_for(ncols * 32, kThreads), kThreads, 0, s, col0, ncols, a.ptr.get(), a.row.get(),
              a.val.get(), dcco.get(), dct.get(), dcc.get(), D);
  if (ne <= 0) return;
  if (ne >= (i64{1} << 31)) fail(PMMF_INTERNAL, "gram: cluster batch exceeds 2^31 entries");
  // Segment bounds (entry ranges of each cluster, relative to e0).
  const i64 nseg = u1 - u0;
  DBuf<int64_t> dseg(nseg + 1, s);
  {
    std::vector<int64_t> cols(static_cast<size_t>(nseg + 1));
    for (i64 u = u0; u <= u1; ++u) cols[u - u0] = off[u];
    DBuf<int64_t> dcols(nseg + 1, s);
    dcols.upload(cols);
    PMMF_LAUNCH(k_gather_ptr, blocks_for(nseg + 1, kThreads), kThreads, 0, s, nseg + 1, dcols.get(), a.ptr.get(), e0,
                dseg.get());
  }
  DBuf<uint64_t> keys(ne, s), keys2(ne, s);
  DBuf<uint32_t> idx(ne, s), idx2(ne, s);
  PMMF_LAUNCH(k_gram_keys, blocks_for(ncols * 32, kThreads), kThreads, 0, s, e0, ne, a.ptr.get(), col0, ncols,
              a.row.get(), dcco.get(), keys.get(), idx.get());
  {
    size_t tmp = 0;
    PMMF_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, tmp, keys.get(), keys2.get(), idx.get(), idx2.get(),
                                                  static_cast<int64_t>(ne), static_cast<int64_t>(nseg), dseg.get(),
                                                  dseg.get() + 1, s));
    DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
    PMMF_CUDA(cub::DeviceSegmentedSort::SortPairs(t.get(), tmp, keys.get(), keys2.get(), idx.get(), idx2.get(),
                                                  static_cast<int64_t>(ne), static_cast<int64_t>(nseg), dseg.get(),
                                                  dseg.get() + 1, s));
  }
  keys.release();
  idx.release();
  DBuf<int64_t> seg_of(ne, s);
  PMMF_LAUNCH(k_seg_of, blocks_for(ne, kThreads), kThreads, 0, s, ne, dseg.get(), nseg, seg_of.get());
  DBuf<int32_t> run_lo(ne, s), run_hi(ne, s), csr_col(ne, s);
  DBuf<double> csr_val(ne, s);
  PMMF_LAUNCH(k_runs, blocks_for(ne, kThreads), kThreads, 0, s, ne, keys2.get(), idx2.get(), seg_of.get(), dseg.get(),
              dseg.get() + 1, a.val.get() + e0, run_lo.get(), run_hi.get(), csr_col.get(), csr_val.get());
  PMMF_LAUNCH(k_gram_owner, blocks_for(ncols * 32, kThreads), kThreads, 0, s, col0, ncols, e0, a.ptr.get(),
              a.val.get(), run_lo.get(), run_hi.get(), csr_col.get(), csr_val.get(), dcco.get(), dct.get(), dcc.get(), G);
  if (trace_enabled()) {  // products = sum over entries of their row-run length (the reference's count)
    DBuf<unsigned long long> tot(1, s);
    tot.zero();
    PMMF_LAUNCH(k_run_total, blocks_for(ne, kThreads), kThreads, 0, s, ne, run_lo.get(), run_hi.get(), tot.get());
    std::fprintf(stderr, "[pmmf]   gram: %lld columns, %lld entries, %llu products\n", static_cast<long long>(ncols),
                 static_cast<long long>(ne), tot.to_host(1)[0]);
  }
}

}  // namespace pmmf_b200
