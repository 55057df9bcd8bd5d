// shard.cu — multi-GPU plumbing of the sharded stage loop (shard.cuh):
// the cluster split, the in-place segment broadcasts over NCCL and the
// gather of the per-rank column slabs; plus the communicator half of the
// C-ABI.  The reference runs the independent clusters of a stage on a
// fork-join thread pool (parallel.hpp:25-71, factorizer.hpp:494-504 and
// :513); here they run on W GPUs.
#include <cub/cub.cuh>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>

#include "shard.cuh"

namespace pmmf_b200 {

namespace {

constexpr int kThreads = 256;
// rotation passes per stored entry vs. Gram/search per tile element: the
// column-pass output of an entry is re-read by the transpose and the row
// pass, and a cluster's tile (c^2) is built once and searched ~c/2 times
// over O(c) rows; fitted on config 4's phase split (apply ~ 2.3x gram+search)
constexpr i64 kApplyWeight = 64;

#define PMMF_NCCL(call)                                                                      \
  do {                                                                                       \
    ncclResult_t r_ = (call);                                                                \
    if (r_ != ncclSuccess)                                                                   \
      ::pmmf_b200::fail(PMMF_CUDA, std::string(#call) + ": " + ncclGetErrorString(r_) + " (" + \
                                       __FILE__ + ":" + std::to_string(__LINE__) + ")");     \
  } while (0)

__global__ void k_gather_i64(i64 n, const i64* __restrict__ src, const i64* __restrict__ idx, i64* __restrict__ dst) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

__global__ void k_ptr_shift(i64 n, const i64* __restrict__ src, i64 sub, i64 add, i64* __restrict__ dst) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < n) dst[i] = src[i] - sub + add;
}

// lens[c - c0] = a.ptr[c+1] - a.ptr[c] for c in [c0, c1)
__global__ void k_col_lens(i64 n, const i64* __restrict__ ptr, i64 c0, int32_t* __restrict__ lens) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < n) lens[i] = static_cast<int32_t>(ptr[c0 + i + 1] - ptr[c0 + i]);
}
__global__ void k_add_lens(i64 n, const int32_t* __restrict__ a, i64* __restrict__ acc) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < n) acc[i] += a[i];
}
// full-width ptr from lengths over [c0, c0+n): ptr[c] = 0 for c <= c0,
// prefix inside, total after
__global__ void k_ptr_fill(i64 N, i64 c0, i64 n, const i64* __restrict__ pre, i64 total, i64* __restrict__ ptr) {
  const i64 c = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (c > N) return;
  ptr[c] = c <= c0 ? 0 : (c >= c0 + n ? total : pre[c - c0]);
}
// warp per column of [c0, c0+n): copy the source's entries of that column
// (source packed in column order, src_off = prefix of its lengths) to dst
__global__ void k_copy_cols(i64 n, i64 c0, const int32_t* __restrict__ lens, const i64* __restrict__ src_off,
                            const int32_t* __restrict__ srow, const double* __restrict__ sval,
                            const i64* __restrict__ dptr, int32_t* __restrict__ drow, double* __restrict__ dval) {
  const i64 w = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  const int len = lens[w];
  if (len == 0) return;
  const i64 so = src_off[w], d0 = dptr[c0 + w];
  for (int e = lane; e < len; e += 32) {
    drow[d0 + e] = srow[so + e];
    dval[d0 + e] = sval[so + e];
  }
}
// anchors: lens of the owned ones
__global__ void k_owned_lens(int m, const int32_t* __restrict__ cols, const i64* __restrict__ ptr, i64 c0, i64 c1,
                             i64* __restrict__ lens) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= m) return;
  const i64 c = cols[a];
  if (c >= c0 && c < c1) lens[a] = ptr[c + 1] - ptr[c];
}
__global__ void k_owned_copy(int m, const int32_t* __restrict__ cols, const i64* __restrict__ ptr,
                             const int32_t* __restrict__ row, const double* __restrict__ val, i64 c0, i64 c1,
                             const i64* __restrict__ off, int32_t* __restrict__ orow, double* __restrict__ oval) {
  const i64 w = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= m) return;
  const i64 c = cols[w];
  if (c < c0 || c >= c1) return;
  const i64 b = ptr[c], n = ptr[c + 1] - b, o = off[w];
  for (i64 e = lane; e < n; e += 32) {
    orow[o + e] = row[b + e];
    oval[o + e] = val[b + e];
  }
}
// column lengths of a gathered set: len[cols[a]] = lens[a]
__global__ void k_scatter_len(int m, const int32_t* __restrict__ cols, const i64* __restrict__ lens,
                              i64* __restrict__ clen) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a < m) clen[cols[a]] = lens[a];
}
__global__ void k_place_cols(int m, const int32_t* __restrict__ cols, const i64* __restrict__ lens,
                             const i64* __restrict__ off, const int32_t* __restrict__ grow,
                             const double* __restrict__ gval, const i64* __restrict__ ptr, int32_t* __restrict__ row,
                             double* __restrict__ val) {
  const i64 w = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= m) return;
  const i64 n = lens[w], o = off[w], d = ptr[cols[w]];
  for (i64 e = lane; e < n; e += 32) {
    row[d + e] = grow[o + e];
    val[d + e] = gval[o + e];
  }
}
// merge: lengths = a's if non-empty else b's
__global__ void k_merge_lens(i64 N, const i64* __restrict__ pa, const i64* __restrict__ pb, i64* __restrict__ len) {
  const i64 c = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (c >= N) return;
  const i64 la = pa[c + 1] - pa[c];
  len[c] = la > 0 ? la : pb[c + 1] - pb[c];
}
__global__ void k_merge_copy(i64 N, const i64* __restrict__ pa, const int32_t* __restrict__ ra,
                             const double* __restrict__ va, const i64* __restrict__ pb, const int32_t* __restrict__ rb,
                             const double* __restrict__ vb, const i64* __restrict__ po, int32_t* __restrict__ ro,
                             double* __restrict__ vo) {
  const i64 w = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= N) return;
  const bool fa = pa[w + 1] > pa[w];
  const i64* p = fa ? pa : pb;
  const int32_t* r = fa ? ra : rb;
  const double* v = fa ? va : vb;
  const i64 b = p[w], n = p[w + 1] - b, d = po[w];
  for (i64 e = lane; e < n; e += 32) {
    ro[d + e] = r[b + e];
    vo[d + e] = v[b + e];
  }
}

template <typename T>
void exscan_dev(const T* in, T* out, i64 n, cudaStream_t s) {
  size_t tmp = 0;
  PMMF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, static_cast<int64_t>(n), s));
  DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
  PMMF_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, in, out, static_cast<int64_t>(n), s));
}

// out (full width) from per-column lengths len[0..N) (int64, device)
void csc_from_lens(Csc& out, const DBuf<i64>& len, i64 N, cudaStream_t s) {
  out = Csc();
  out.N = N;
  out.ptr.alloc(N + 1, s);
  DBuf<i64> l1(N + 1, s);
  PMMF_CUDA(cudaMemsetAsync(l1.get() + N, 0, sizeof(i64), s));
  if (N) PMMF_CUDA(cudaMemcpyAsync(l1.get(), len.get(), sizeof(i64) * N, cudaMemcpyDeviceToDevice, s));
  exscan_dev(l1.get(), out.ptr.get(), N + 1, s);
  out.nnz = out.ptr.to_host(N + 1)[N];
  out.row.alloc(std::max<i64>(out.nnz, 1), s);
  out.val.alloc(std::max<i64>(out.nnz, 1), s);
}

}  // namespace

void allreduce_sum_i64(int64_t* dev, i64 n, const Comm& c, cudaStream_t s) {
  if (!c.multi_process() || n <= 0) return;
  PMMF_NCCL(ncclAllReduce(dev, dev, static_cast<size_t>(n), ncclInt64, ncclSum, c.nccl, s));
}
void allreduce_sum_f64(double* dev, i64 n, const Comm& c, cudaStream_t s) {
  if (!c.multi_process() || n <= 0) return;
  PMMF_NCCL(ncclAllReduce(dev, dev, static_cast<size_t>(n), ncclFloat64, ncclSum, c.nccl, s));
}
void allreduce_max_f64(double* dev, i64 n, const Comm& c, cudaStream_t s) {
  if (!c.multi_process() || n <= 0) return;
  PMMF_NCCL(ncclAllReduce(dev, dev, static_cast<size_t>(n), ncclFloat64, ncclMax, c.nccl, s));
}

void slab_of(Csc& out, const Csc& a, i64 c0, i64 c1, cudaStream_t s) {
  const i64 N = a.N, n = std::max<i64>(c1 - c0, 0);
  DBuf<i64> len(std::max<i64>(N, 1), s);
  len.zero();
  {
    DBuf<int32_t> l32(std::max<i64>(n, 1), s);
    PMMF_LAUNCH(k_col_lens, blocks_for(n, kThreads), kThreads, 0, s, n, a.ptr.get(), c0, l32.get());
    PMMF_LAUNCH(k_add_lens, blocks_for(n, kThreads), kThreads, 0, s, n, l32.get(), len.get() + c0);
  }
  csc_from_lens(out, len, N, s);
  if (out.nnz > 0) {
    i64 b = 0;
    PMMF_CUDA(cudaMemcpyAsync(&b, a.ptr.get() + c0, sizeof(i64), cudaMemcpyDeviceToHost, s));
    PMMF_CUDA(cudaStreamSynchronize(s));
    PMMF_CUDA(cudaMemcpyAsync(out.row.get(), a.row.get() + b, sizeof(int32_t) * out.nnz, cudaMemcpyDeviceToDevice, s));
    PMMF_CUDA(cudaMemcpyAsync(out.val.get(), a.val.get() + b, sizeof(double) * out.nnz, cudaMemcpyDeviceToDevice, s));
  }
}

void gather_columns(Csc& out, const std::vector<const Csc*>& slabs, const std::vector<std::pair<i64, i64>>& own,
                    const int32_t* cols, int m, i64 N, const Comm& c, cudaStream_t s) {
  DBuf<i64> lens(std::max(m, 1), s), off(std::max(m, 1) + 1, s);
  lens.zero();
  for (size_t i = 0; i < slabs.size(); ++i)
    PMMF_LAUNCH(k_owned_lens, blocks_for(m, kThreads), kThreads, 0, s, m, cols, slabs[i]->ptr.get(), own[i].first,
                own[i].second, lens.get());
  allreduce_sum_i64(lens.get(), m, c, s);
  {
    DBuf<i64> l1(m + 1, s);
    PMMF_CUDA(cudaMemsetAsync(l1.get() + m, 0, sizeof(i64), s));
    if (m) PMMF_CUDA(cudaMemcpyAsync(l1.get(), lens.get(), sizeof(i64) * m, cudaMemcpyDeviceToDevice, s));
    exscan_dev(l1.get(), off.get(), m + 1, s);
  }
  const i64 total = off.to_host(m + 1)[m];
  DBuf<int32_t> grow(std::max<i64>(total, 1), s);
  DBuf<double> gval(std::max<i64>(total, 1), s);
  if (c.multi_process()) {  // every entry owned by one rank: zeros elsewhere, then sums
    grow.zero();
    gval.zero();
  }
  for (size_t i = 0; i < slabs.size(); ++i)
    PMMF_LAUNCH(k_owned_copy, blocks_for(static_cast<i64>(m) * 32, kThreads), kThreads, 0, s, m, cols,
                slabs[i]->ptr.get(), slabs[i]->row.get(), slabs[i]->val.get(), own[i].first, own[i].second, off.get(),
                grow.get(), gval.get());
  if (c.multi_process() && total > 0) {
    PMMF_NCCL(ncclAllReduce(grow.get(), grow.get(), static_cast<size_t>(total), ncclInt32, ncclSum, c.nccl, s));
    allreduce_sum_f64(gval.get(), total, c, s);
  }
  DBuf<i64> clen(std::max<i64>(N, 1), s);
  clen.zero();
  PMMF_LAUNCH(k_scatter_len, blocks_for(m, kThreads), kThreads, 0, s, m, cols, lens.get(), clen.get());
  csc_from_lens(out, clen, N, s);
  PMMF_LAUNCH(k_place_cols, blocks_for(static_cast<i64>(m) * 32, kThreads), kThreads, 0, s, m, cols, lens.get(),
              off.get(), grow.get(), gval.get(), out.ptr.get(), out.row.get(), out.val.get());
}

void merge_columns(Csc& out, const Csc& a, const Csc& b, cudaStream_t s) {
  const i64 N = a.N;
  DBuf<i64> len(std::max<i64>(N, 1), s);
  PMMF_LAUNCH(k_merge_lens, blocks_for(N, kThreads), kThreads, 0, s, N, a.ptr.get(), b.ptr.get(), len.get());
  csc_from_lens(out, len, N, s);
  PMMF_LAUNCH(k_merge_copy, blocks_for(N * 32, kThreads), kThreads, 0, s, N, a.ptr.get(), a.row.get(), a.val.get(),
              b.ptr.get(), b.row.get(), b.val.get(), out.ptr.get(), out.row.get(), out.val.get());
}

void redistribute(std::vector<Csc>& slabs, const std::vector<i64>& dest, i64 N, const Comm& c, cudaStream_t s) {
  const std::vector<int> mine = c.local_ranks();
  const int W = c.size;
  if (!c.multi_process()) {
    // virtual ranks (or one): every destination slab from every local source
    std::vector<Csc> out(mine.size());
    for (size_t di = 0; di < mine.size(); ++di) {
      const int d = mine[di];
      const i64 c0 = dest[d], n = dest[d + 1] - dest[d];
      DBuf<i64> len(std::max<i64>(N, 1), s);
      len.zero();
      std::vector<DBuf<int32_t>> sl(slabs.size());
      for (size_t si = 0; si < slabs.size(); ++si) {
        sl[si].alloc(std::max<i64>(n, 1), s);
        PMMF_LAUNCH(k_col_lens, blocks_for(n, kThreads), kThreads, 0, s, n, slabs[si].ptr.get(), c0, sl[si].get());
        PMMF_LAUNCH(k_add_lens, blocks_for(n, kThreads), kThreads, 0, s, n, sl[si].get(), len.get() + c0);
      }
      csc_from_lens(out[di], len, N, s);
      for (size_t si = 0; si < slabs.size(); ++si) {
        // the source's entries of [c0, c0+n) are contiguous from ptr[c0]
        DBuf<i64> so(std::max<i64>(n, 1), s);
        PMMF_LAUNCH(k_ptr_shift, blocks_for(n, kThreads), kThreads, 0, s, n, slabs[si].ptr.get() + c0, i64{0}, i64{0},
                    so.get());
        PMMF_LAUNCH(k_copy_cols, blocks_for(n * 32, kThreads), kThreads, 0, s, n, c0, sl[si].get(), so.get(),
                    slabs[si].row.get(), slabs[si].val.get(), out[di].ptr.get(), out[di].row.get(),
                    out[di].val.get());
      }
    }
    slabs = std::move(out);
    return;
  }
  // one local rank per process: counts, lengths and entries by ncclSend/Recv
  const int me = c.rank;
  Csc& B = slabs[0];
  std::vector<i64> at(static_cast<size_t>(W) + 1);
  {
    DBuf<i64> idx(W + 1, s), v(W + 1, s);
    idx.upload(dest);
    PMMF_LAUNCH(k_gather_i64, blocks_for(W + 1, kThreads), kThreads, 0, s, W + 1, B.ptr.get(), idx.get(), v.get());
    at = v.to_host(W + 1);
  }
  // counts[s * W + d] = entries rank s sends to rank d
  DBuf<i64> dcnt(static_cast<i64>(W) * W, s);
  {
    std::vector<i64> mycnt(static_cast<size_t>(W));
    for (int d = 0; d < W; ++d) mycnt[d] = at[d + 1] - at[d];
    DBuf<i64> sendc(W, s);
    sendc.upload(mycnt);
    PMMF_NCCL(ncclAllGather(sendc.get(), dcnt.get(), static_cast<size_t>(W), ncclInt64, c.nccl, s));
  }
  const std::vector<i64> cnt = dcnt.to_host(static_cast<i64>(W) * W);
  const i64 c0 = dest[me], n = dest[me + 1] - dest[me];
  // my lengths per destination range, and receive buffers per source
  std::vector<DBuf<int32_t>> send_len(static_cast<size_t>(W)), recv_len(static_cast<size_t>(W)), recv_row(static_cast<size_t>(W));
  std::vector<DBuf<double>> recv_val(static_cast<size_t>(W));
  for (int d = 0; d < W; ++d) {
    const i64 nd = dest[d + 1] - dest[d];
    send_len[d].alloc(std::max<i64>(nd, 1), s);
    PMMF_LAUNCH(k_col_lens, blocks_for(nd, kThreads), kThreads, 0, s, nd, B.ptr.get(), dest[d], send_len[d].get());
  }
  for (int src = 0; src < W; ++src) {
    recv_len[src].alloc(std::max<i64>(n, 1), s);
    const i64 k = cnt[static_cast<size_t>(src) * W + me];
    recv_row[src].alloc(std::max<i64>(k, 1), s);
    recv_val[src].alloc(std::max<i64>(k, 1), s);
  }
  PMMF_NCCL(ncclGroupStart());
  for (int d = 0; d < W; ++d) {
    const i64 nd = dest[d + 1] - dest[d], k = at[d + 1] - at[d];
    if (nd > 0) PMMF_NCCL(ncclSend(send_len[d].get(), static_cast<size_t>(nd), ncclInt32, d, c.nccl, s));
    if (k > 0) {
      PMMF_NCCL(ncclSend(B.row.get() + at[d], static_cast<size_t>(k), ncclInt32, d, c.nccl, s));
      PMMF_NCCL(ncclSend(B.val.get() + at[d], static_cast<size_t>(k), ncclFloat64, d, c.nccl, s));
    }
  }
  for (int src = 0; src < W; ++src) {
    const i64 k = cnt[static_cast<size_t>(src) * W + me];
    if (n > 0) PMMF_NCCL(ncclRecv(recv_len[src].get(), static_cast<size_t>(n), ncclInt32, src, c.nccl, s));
    if (k > 0) {
      PMMF_NCCL(ncclRecv(recv_row[src].get(), static_cast<size_t>(k), ncclInt32, src, c.nccl, s));
      PMMF_NCCL(ncclRecv(recv_val[src].get(), static_cast<size_t>(k), ncclFloat64, src, c.nccl, s));
    }
  }
  PMMF_NCCL(ncclGroupEnd());
  DBuf<i64> len(std::max<i64>(N, 1), s);
  len.zero();
  for (int src = 0; src < W; ++src)
    PMMF_LAUNCH(k_add_lens, blocks_for(n, kThreads), kThreads, 0, s, n, recv_len[src].get(), len.get() + c0);
  Csc out;
  csc_from_lens(out, len, N, s);
  for (int src = 0; src < W; ++src) {
    DBuf<i64> l64(std::max<i64>(n, 1) + 1, s), so(std::max<i64>(n, 1) + 1, s);
    l64.zero();
    PMMF_LAUNCH(k_add_lens, blocks_for(n, kThreads), kThreads, 0, s, n, recv_len[src].get(), l64.get());
    exscan_dev(l64.get(), so.get(), n + 1, s);
    PMMF_LAUNCH(k_copy_cols, blocks_for(n * 32, kThreads), kThreads, 0, s, n, c0, recv_len[src].get(), so.get(),
                recv_row[src].get(), recv_val[src].get(), out.ptr.get(), out.row.get(), out.val.get());
  }
  slabs[0] = std::move(out);
  PMMF_CUDA(cudaStreamSynchronize(s));
}

std::vector<i64> shard_ranges(const std::vector<i64>& size, const std::vector<i64>& nnz, int W) {
  const i64 m = static_cast<i64>(size.size());
  W = std::max(W, 1);
  std::vector<i64> lo(static_cast<size_t>(W) + 1, m);
  lo[0] = 0;
  std::vector<double> pre(static_cast<size_t>(m) + 1, 0.0);
  for (i64 u = 0; u < m; ++u) {
    const double c = static_cast<double>(size[u]);
    const double z = u < static_cast<i64>(nnz.size()) ? static_cast<double>(nnz[u]) : 0.0;
    pre[u + 1] = pre[u] + c * c + static_cast<double>(kApplyWeight) * z;
  }
  // boundary r: the first cluster whose cost prefix reaches r/W of the total
  // (monotone, so the ranges are contiguous; empty ranges allowed)
  i64 u = 0;
  for (int r = 1; r < W; ++r) {
    const double target = pre[m] * static_cast<double>(r) / static_cast<double>(W);
    while (u < m && pre[u + 1] <= target) ++u;
    // put cluster u on the side that leaves the prefix closer to the target
    i64 b = u;
    if (u < m && target - pre[u] > pre[u + 1] - target) b = u + 1;
    lo[r] = std::max(b, lo[r - 1]);
  }
  lo[W] = m;
  return lo;
}

std::vector<i64> cluster_ptr(const Csc& a, const std::vector<i64>& off, cudaStream_t s) {
  const i64 m = static_cast<i64>(off.size());
  if (m == 0) return {};
  DBuf<i64> idx(m, s), out(m, s);
  idx.upload(off);
  PMMF_LAUNCH(k_gather_i64, blocks_for(m, kThreads), kThreads, 0, s, m, a.ptr.get(), idx.get(), out.get());
  return out.to_host(m);
}

void bcast_segments(void* dev, size_t elem, const std::vector<i64>& seg, const Comm& c, cudaStream_t s) {
  if (!c.multi_process()) return;
  auto* base = static_cast<char*>(dev);
  PMMF_NCCL(ncclGroupStart());
  for (int r = 0; r < c.size; ++r) {
    const i64 n = seg[r + 1] - seg[r];
    if (n <= 0) continue;
    char* p = base + static_cast<size_t>(seg[r]) * elem;
    PMMF_NCCL(ncclBroadcast(p, p, static_cast<size_t>(n) * elem, ncclChar, r, c.nccl, s));
  }
  PMMF_NCCL(ncclGroupEnd());
}

void allreduce_max_i32(int32_t* dev, const Comm& c, cudaStream_t s) { allreduce_max_i32(dev, 1, c, s); }

void allreduce_max_i32(int32_t* dev, i64 n, const Comm& c, cudaStream_t s) {
  if (!c.multi_process() || n <= 0) return;
  PMMF_NCCL(ncclAllReduce(dev, dev, static_cast<size_t>(n), ncclInt32, ncclMax, c.nccl, s));
}

}  // namespace pmmf_b200

// ---- C-ABI (include/pmmf_b200.h, multi-GPU section)

using namespace pmmf_b200;

namespace pmmf_b200 {
int guarded_call(char* err, size_t errlen, void (*fn)(void*), void* ctx);
}

template <typename F>
static int guarded(char* err, size_t errlen, F&& f) {
  return guarded_call(err, errlen, [](void* c) { (*static_cast<F*>(c))(); }, &f);
}

extern "C" {

int pmmf_b200_comm_unique_id(uint8_t* id, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!id) fail(PMMF_INVALID_ARGUMENT, "pmmf_b200_comm_unique_id: null argument");
    static_assert(sizeof(ncclUniqueId) == PMMF_B200_COMM_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId u;
    PMMF_NCCL(ncclGetUniqueId(&u));
    std::memcpy(id, &u, sizeof(u));
  });
}

int pmmf_b200_comm_create(int32_t nranks, int32_t rank, const uint8_t* id, int32_t device, void** comm, char* err,
                          size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!comm || (!id && nranks > 1)) fail(PMMF_INVALID_ARGUMENT, "pmmf_b200_comm_create: null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(PMMF_INVALID_ARGUMENT, "pmmf_b200_comm_create: bad rank");
    auto c = std::make_unique<Comm>();
    c->rank = rank;
    c->size = nranks;
    c->device = device;
    {
      PMMF_CUDA(cudaSetDevice(device));
      ncclUniqueId u;
      if (id) {
        std::memcpy(&u, id, sizeof(u));
      } else {
        PMMF_NCCL(ncclGetUniqueId(&u));
      }
      ncclComm_t nc = nullptr;
      PMMF_NCCL(ncclCommInitRank(&nc, nranks, u, rank));
      c->nccl = nc;
    }
    *comm = c.release();
  });
}

int pmmf_b200_comm_create_virtual(int32_t nranks, int32_t device, void** comm, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!comm) fail(PMMF_INVALID_ARGUMENT, "pmmf_b200_comm_create_virtual: null argument");
    if (nranks < 1) fail(PMMF_INVALID_ARGUMENT, "pmmf_b200_comm_create_virtual: nranks < 1");
    auto c = std::make_unique<Comm>();
    c->size = nranks;
    c->virt = true;
    c->device = device;
    *comm = c.release();
  });
}

void pmmf_b200_comm_free(void* comm) {
  auto* c = static_cast<Comm*>(comm);
  if (!c) return;
  if (c->nccl) ncclCommDestroy(c->nccl);
  delete c;
}

int pmmf_b200_shard_ranges(int64_t nclusters, const int64_t* sizes, const int64_t* nnz, int32_t nranks,
                           int64_t* lo) {
  if (nclusters < 0 || nranks < 1 || (!sizes && nclusters) || !lo) return PMMF_INVALID_ARGUMENT;
  std::vector<i64> sz(sizes, sizes + nclusters), z;
  if (nnz) z.assign(nnz, nnz + nclusters);
  const std::vector<i64> r = shard_ranges(sz, z, nranks);
  std::copy(r.begin(), r.end(), lo);
  return PMMF_OK;
}

}  // extern "C"
