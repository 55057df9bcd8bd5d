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
  // One stable radix sort on (cluster index in the batch, row) keeps the
  // columns ascending inside a run; a run is a row's entries inside the
  // owner column's own cluster.
  const i64 N = a.N;
  const i64 nseg = u1 - u0;
  const int rb = std::max(1, bits_for(std::max<i64>(N - 1, 1)));
  const int sb = std::max(1, bits_for(std::max<i64>(nseg - 1, 1)));
  std::vector<int32_t> seg(static_cast<size_t>(ncols));
  for (i64 u = u0; u < u1; ++u)
    for (i64 J = off[u]; J < off[u + 1]; ++J) seg[J - col0] = static_cast<int32_t>(u - u0);
  DBuf<int32_t> dseg(ncols, s);
  dseg.upload(seg);
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
