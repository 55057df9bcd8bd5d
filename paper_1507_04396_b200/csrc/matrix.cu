// matrix.cu — blocked-matrix plumbing of the stage loop on the device:
// from_triplets, symmetry check, paged<->contiguous transposes and reblock.
// All of it is HBM-bound integer/byte movement: coalesced warp-per-column
// gathers plus CUB radix / segmented sorts (row-key only, so the sorts run
// over ceil(log2 N)/8 digit passes, not a full 64-bit key).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>

#include "engine.cuh"

namespace pmmf_b200 {

namespace {
double ms_since_tp(std::chrono::steady_clock::time_point t) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
}
}  // namespace

namespace {

constexpr int kThreads = 256;

// ------------------------------------------------------------ numbering
__global__ void k_fill_blk(const int64_t* off, i64 m, int32_t* blk) {
  const i64 u = blockIdx.x;
  if (u >= m) return;
  for (i64 i = off[u] + threadIdx.x; i < off[u + 1]; i += blockDim.x) blk[i] = static_cast<int32_t>(u);
}

// ------------------------------------------------------------ from_coo
__global__ void k_g2s(i64 N, const int32_t* __restrict__ s2g, int32_t* __restrict__ g2s) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < N) g2s[s2g[i]] = static_cast<int32_t>(i);
}

__global__ void k_coo_keys(i64 n, i64 nnz, const int64_t* __restrict__ rows, const int64_t* __restrict__ cols,
                           const double* __restrict__ vals, const int32_t* __restrict__ g2s, uint64_t N,
                           uint64_t* __restrict__ keys, unsigned long long* __restrict__ first_err) {
  const i64 t = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (t >= nnz) return;
  const i64 r = rows[t], c = cols[t];
  const double v = vals[t];
  unsigned code = 0;
  i64 sr = -1, sc = -1;
  if (r < 0 || r >= n || c < 0 || c >= n) {
    code = 1;  // out_of_range: index out of range
  } else if (!isfinite(v)) {
    code = 2;  // invalid_argument: non-finite value
  } else {
    sr = g2s[r];
    sc = g2s[c];
    if (sr < 0 || sc < 0) code = 3;  // out_of_range: not covered
  }
  if (code) {
    atomicMin(first_err, (static_cast<unsigned long long>(t) << 2) | code);
    keys[t] = 0;
    return;
  }
  keys[t] = static_cast<uint64_t>(sc) * N + static_cast<uint64_t>(sr);
}

// Sum runs of equal keys in their (stable) order; flag the kept heads.
__global__ void k_sum_dups(i64 m, const uint64_t* __restrict__ keys, const double* __restrict__ vals,
                           double* __restrict__ sums, int32_t* __restrict__ keep, bool keep_zeros) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= m) return;
  if (i > 0 && keys[i - 1] == keys[i]) {
    keep[i] = 0;
    return;
  }
  double s = vals[i];
  for (i64 j = i + 1; j < m && keys[j] == keys[i]; ++j) s = dadd(s, vals[j]);
  sums[i] = s;
  keep[i] = (keep_zeros || s != 0.0) ? 1 : 0;
}

__global__ void k_scatter_kept(i64 m, const uint64_t* __restrict__ keys, const double* __restrict__ sums,
                               const int32_t* __restrict__ keep, const i64* __restrict__ pos, uint64_t N,
                               int32_t* __restrict__ out_col, int32_t* __restrict__ out_row,
                               double* __restrict__ out_val) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= m || !keep[i]) return;
  const i64 p = pos[i];
  out_col[p] = static_cast<int32_t>(keys[i] / N);
  out_row[p] = static_cast<int32_t>(keys[i] % N);
  out_val[p] = sums[i];
}

// ptr[c] = first position whose column >= c, for a column-sorted list.
__global__ void k_ptr_from_cols(i64 m, const int32_t* __restrict__ col, i64 N, i64* __restrict__ ptr) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i > m) return;
  const i64 prev = i == 0 ? -1 : col[i - 1];
  const i64 cur = i == m ? N : col[i];
  for (i64 c = prev + 1; c <= cur; ++c) ptr[c] = i;
}

// ---------------------------------------------------------- symmetry
__global__ void k_symmetry(i64 N, const i64* __restrict__ ptr, const int32_t* __restrict__ row,
                           const double* __restrict__ val, const int32_t* __restrict__ blk,
                           unsigned long long* __restrict__ worst, double* __restrict__ col_fro) {
  // warp per column (hub columns of R-MAT inputs hold 10^4-10^5 entries);
  // the Frobenius sum only feeds the 1e-9 threshold, so its order is free.
  const i64 j = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= N) return;
  double fro = 0.0, w = 0.0;
  const int32_t bj = blk[j];
  for (i64 e = ptr[j] + lane; e < ptr[j + 1]; e += 32) {
    const double v = val[e];
    fro = dadd(fro, dmul(v, v));
    const int32_t r = row[e];
    if (blk[r] > bj) continue;
    // mirror value A[j][r]: row j of column r
    i64 lo = ptr[r], hi = ptr[r + 1];
    while (lo < hi) {
      const i64 mid = (lo + hi) >> 1;
      if (row[mid] < j) lo = mid + 1; else hi = mid;
    }
    const double mv = (lo < ptr[r + 1] && row[lo] == j) ? val[lo] : 0.0;
    w = fmax(w, fabs(dsub(v, mv)));
  }
  for (int o = 16; o; o >>= 1) {
    fro = dadd(fro, __shfl_xor_sync(0xffffffffu, fro, o));
    w = fmax(w, __shfl_xor_sync(0xffffffffu, w, o));
  }
  if (lane != 0) return;
  col_fro[j] = fro;
  if (w > 0.0) atomicMax(worst, static_cast<unsigned long long>(__double_as_longlong(w)));
}

// ----------------------------------------------------------- paged
__global__ void k_paged_init(i64 N, const i64* __restrict__ ptr, i64* __restrict__ off, int32_t* __restrict__ len) {
  const i64 j = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (j >= N) return;
  off[j] = ptr[j];
  len[j] = static_cast<int32_t>(ptr[j + 1] - ptr[j]);
}

__global__ void k_len64(i64 N, const int32_t* __restrict__ len, i64* __restrict__ out) {
  const i64 j = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (j < N) out[j] = len[j];
  if (j == N) out[j] = 0;
}

// Gather the paged columns in column order into (row<<cb | col, val).
__global__ void k_gather_keys(i64 N, const i64* __restrict__ off, const int32_t* __restrict__ len,
                              const int32_t* __restrict__ arow, const double* __restrict__ aval,
                              const i64* __restrict__ pos, int cb, uint64_t* __restrict__ keys,
                              double* __restrict__ vals) {
  const i64 warp = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= N) return;
  const i64 src = off[warp], dst = pos[warp];
  const int32_t L = len[warp];
  for (int32_t i = lane; i < L; i += 32) {
    keys[dst + i] = (static_cast<uint64_t>(arow[src + i]) << cb) | static_cast<uint64_t>(warp);
    vals[dst + i] = aval[src + i];
  }
}

__global__ void k_split_keys(i64 m, const uint64_t* __restrict__ keys, int cb, int32_t* __restrict__ major,
                             int32_t* __restrict__ minor) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= m) return;
  const uint64_t k = keys[i];
  major[i] = static_cast<int32_t>(k >> cb);
  minor[i] = static_cast<int32_t>(k & ((uint64_t{1} << cb) - 1));
}

// ----------------------------------------------------------- reblock
__global__ void k_reblock_count(i64 Nn, const int32_t* __restrict__ new2old, const i64* __restrict__ ptr,
                                const int32_t* __restrict__ row, const int32_t* __restrict__ map,
                                i64* __restrict__ cnt) {
  const i64 warp = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp > Nn) return;
  if (warp == Nn) {
    if (lane == 0) cnt[Nn] = 0;
    return;
  }
  const int32_t j = new2old[warp];
  int c = 0;
#pragma unroll 4
  for (i64 e = ptr[j] + lane; e < ptr[j + 1]; e += 32) c += map[row[e]] >= 0;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) cnt[warp] = c;
}

__global__ void k_reblock_fill(i64 Nn, const int32_t* __restrict__ new2old, const i64* __restrict__ ptr,
                               const int32_t* __restrict__ row, const double* __restrict__ val,
                               const int32_t* __restrict__ map, const i64* __restrict__ nptr,
                               int32_t* __restrict__ nrow, double* __restrict__ nval) {
  const i64 warp = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= Nn) return;
  const int32_t j = new2old[warp];
  i64 out = nptr[warp];
  const i64 e1 = ptr[j + 1];
  // four windows per round: the rows, the relabel gathers and the values of all
  // four are in flight together (a hub column is one warp's sequential loop)
  for (i64 base = ptr[j]; base < e1; base += 128) {
    int32_t r[4], nr[4];
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const i64 e = base + 32 * q + lane;
      r[q] = e < e1 ? row[e] : -1;
      v[q] = e < e1 ? val[e] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) nr[q] = r[q] >= 0 ? map[r[q]] : -1;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const unsigned keep = __ballot_sync(0xffffffffu, nr[q] >= 0);
      if (nr[q] >= 0) {
        const int p = __popc(keep & ((1u << lane) - 1));
        nrow[out + p] = nr[q];
        nval[out + p] = v[q];
      }
      out += __popc(keep);
    }
  }
}

// ---------------------------------------------------- chunked transpose
__global__ void k_row_hist(i64 N, const i64* __restrict__ ptr, const int32_t* __restrict__ row,
                           const uint8_t* __restrict__ keep_row, int32_t* __restrict__ hist) {
  const i64 w = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= N) return;
  for (i64 e = ptr[w] + lane; e < ptr[w + 1]; e += 32) {
    const int32_t r = row[e];
    if (keep_row == nullptr || keep_row[r]) atomicAdd(&hist[r], 1);
  }
}
__device__ __forceinline__ i64 lb_rows(const int32_t* __restrict__ a, i64 lo, i64 hi, int key) {
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}
// Entries of piece column w with row in [r0, r1) (and kept by the filter).
__global__ void k_chunk_count(i64 N, i64 c0, const i64* __restrict__ ptr, const int32_t* __restrict__ row,
                              const uint8_t* __restrict__ keep_row, int r0, int r1, i64* __restrict__ cnt) {
  const i64 w = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= N) return;
  const i64 lo = lb_rows(row, ptr[w], ptr[w + 1], r0), hi = lb_rows(row, lo, ptr[w + 1], r1);
  int c = 0;
  if (keep_row == nullptr) {
    c = lane == 0 ? static_cast<int>(hi - lo) : 0;
  } else {
    for (i64 e = lo + lane; e < hi; e += 32) c += keep_row[row[e]];
  }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) cnt[c0 + w] = c;
}
__global__ void k_chunk_gather(i64 N, i64 c0, const i64* __restrict__ ptr, const int32_t* __restrict__ row,
                               const double* __restrict__ val, const uint8_t* __restrict__ keep_row, int r0, int r1,
                               const i64* __restrict__ pos, int cb, uint64_t* __restrict__ keys,
                               double* __restrict__ vals) {
  const i64 w = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= N) return;
  const i64 lo = lb_rows(row, ptr[w], ptr[w + 1], r0), hi = lb_rows(row, lo, ptr[w + 1], r1);
  i64 o = pos[c0 + w];
  const uint64_t col = static_cast<uint64_t>(c0 + w);
  for (i64 b = lo; b < hi; b += 128) {  // four windows per round, loads of all four in flight
    int32_t r[4];
    bool k[4];
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const i64 e = b + 32 * q + lane;
      r[q] = e < hi ? row[e] : -1;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      k[q] = r[q] >= 0 && (keep_row == nullptr || keep_row[r[q]]);
      v[q] = k[q] ? val[b + 32 * q + lane] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const unsigned m = __ballot_sync(0xffffffffu, k[q]);
      if (k[q]) {
        const i64 d = o + __popc(m & ((1u << lane) - 1u));
        keys[d] = (static_cast<uint64_t>(r[q] - r0) << cb) | col;
        vals[d] = v[q];
      }
      o += __popc(m);
    }
  }
}
__global__ void k_chunk_emit(i64 m, const uint64_t* __restrict__ keys, const double* __restrict__ vals, int cb,
                             int32_t* __restrict__ out_row, double* __restrict__ out_val) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= m) return;
  out_row[i] = static_cast<int32_t>(keys[i] & ((uint64_t{1} << cb) - 1));
  out_val[i] = vals[i];
}
__global__ void k_hist_widen(i64 N, const int32_t* __restrict__ h, i64* __restrict__ out) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < N) out[i] = h[i];
  if (i == N) out[i] = 0;
}

template <typename T>
void exclusive_scan(const T* in, T* out, i64 n, cudaStream_t s) {
  size_t tmp = 0;
  PMMF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, static_cast<int64_t>(n), s));
  DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
  PMMF_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, in, out, static_cast<int64_t>(n), s));
}

void sort_pairs(DBuf<uint64_t>& keys, DBuf<double>& vals, i64 m, int begin_bit, int end_bit, cudaStream_t s) {
  if (m <= 1 || end_bit <= begin_bit) return;
  DBuf<uint64_t> k2(m, s);
  DBuf<double> v2(m, s);
  cub::DoubleBuffer<uint64_t> kb(keys.get(), k2.get());
  cub::DoubleBuffer<double> vb(vals.get(), v2.get());
  size_t tmp = 0;
  PMMF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, static_cast<int64_t>(m), begin_bit, end_bit, s));
  DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
  PMMF_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, kb, vb, static_cast<int64_t>(m), begin_bit, end_bit, s));
  if (kb.Current() != keys.get()) {  // whole buffers: a cached block may be larger than requested
    std::swap(keys, k2);
    std::swap(vals, v2);
  }
}

}  // namespace

std::atomic<int64_t>& launch_counter() {
  static std::atomic<int64_t> c{0};
  return c;
}

void Numbering::build(const std::vector<std::vector<i64>>& cls, i64 n, cudaStream_t s) {
  s2g.clear();
  off.assign(1, 0);
  g2s.assign(static_cast<size_t>(std::max<i64>(n, 0)), -1);
  for (const auto& cl : cls) {
    for (i64 g : cl) {
      if (g < 0) fail(PMMF_INVALID_ARGUMENT, "Partition: negative index");
      if (g >= n) fail(PMMF_OUT_OF_RANGE, "Partition: index beyond matrix dimension");
      if (g2s[g] >= 0) fail(PMMF_INVALID_ARGUMENT, "Partition: duplicate index across clusters");
      g2s[g] = static_cast<i64>(s2g.size());
      s2g.push_back(g);
    }
    off.push_back(static_cast<i64>(s2g.size()));
  }
  const i64 N = size();
  d_blk.alloc(std::max<i64>(N, 1), s);
  d_s2g.alloc(std::max<i64>(N, 1), s);
  std::vector<int32_t> s2g32(s2g.begin(), s2g.end());
  d_s2g.upload(s2g32);
  DBuf<int64_t> doff(clusters() + 1, s);
  doff.upload(off);
  PMMF_LAUNCH(k_fill_blk, static_cast<unsigned>(clusters()), 256, 0, s, doff.get(), clusters(), d_blk.get());
  d_g2s.alloc(std::max<i64>(n, 1), s);
  d_g2s.fill_bytes(0xff);
  PMMF_LAUNCH(k_g2s, blocks_for(N, 256), 256, 0, s, N, d_s2g.get(), d_g2s.get());
}

void Numbering::build_device(DBuf<int32_t>&& members, std::vector<i64> offsets, i64 n, cudaStream_t s) {
  off = std::move(offsets);
  const i64 N = off.back();
  d_s2g = std::move(members);
  d_blk.alloc(std::max<i64>(N, 1), s);
  DBuf<int64_t> doff(clusters() + 1, s);
  doff.upload(off);
  PMMF_LAUNCH(k_fill_blk, static_cast<unsigned>(clusters()), 256, 0, s, doff.get(), clusters(), d_blk.get());
  d_g2s.alloc(std::max<i64>(n, 1), s);
  d_g2s.fill_bytes(0xff);
  PMMF_LAUNCH(k_g2s, blocks_for(N, 256), 256, 0, s, N, d_s2g.get(), d_g2s.get());
  // host mirror of stage -> global; global -> stage (n entries whatever the
  // stage's size: ~1.5 ms per stage at n = 2^20) is fetched on demand
  std::vector<int32_t> h = d_s2g.to_host(N);
  s2g.assign(h.begin(), h.end());
  g2s.clear();
  n_global = n;
}

const std::vector<i64>& Numbering::host_g2s() {
  if (g2s.empty() && n_global > 0) {
    std::vector<int32_t> hg = d_g2s.to_host(n_global);
    g2s.assign(hg.begin(), hg.end());
  }
  return g2s;
}

void csc_from_coo(Csc& out, const Numbering& nb, i64 n, i64 nnz, const int64_t* rows, const int64_t* cols,
                  const double* vals, cudaStream_t s, bool keep_zeros) {
  const i64 N = nb.size();
  out.N = N;
  DBuf<int32_t> g2s(std::max<i64>(n, 1), s);
  {
    std::vector<int32_t> h(nb.g2s.begin(), nb.g2s.end());
    g2s.upload(h);
  }
  DBuf<uint64_t> keys(std::max<i64>(nnz, 1), s);
  DBuf<double> v(std::max<i64>(nnz, 1), s);
  DBuf<unsigned long long> ferr(1, s);
  ferr.fill_bytes(0xff);
  if (nnz > 0) {
    PMMF_CUDA(cudaMemcpyAsync(v.get(), vals, sizeof(double) * nnz, cudaMemcpyDeviceToDevice, s));
    PMMF_LAUNCH(k_coo_keys, blocks_for(nnz, kThreads), kThreads, 0, s, n, nnz, rows, cols, vals, g2s.get(),
                static_cast<uint64_t>(std::max<i64>(N, 1)), keys.get(), ferr.get());
  }
  const unsigned long long fe = ferr.to_host(1)[0];
  if (fe != ~0ull) {
    const unsigned code = fe & 3u;
    if (code == 1) fail(PMMF_OUT_OF_RANGE, "from_triplets: index out of range");
    if (code == 2) fail(PMMF_INVALID_ARGUMENT, "from_triplets: non-finite value");
    fail(PMMF_OUT_OF_RANGE, "from_triplets: index not covered by partition");
  }
  const int kb = bits_for(std::max<i64>(N, 1) * std::max<i64>(N, 1) - 1);
  sort_pairs(keys, v, nnz, 0, std::max(kb, 1), s);
  DBuf<double> sums(std::max<i64>(nnz, 1), s);
  DBuf<int32_t> keep(nnz + 1, s);
  DBuf<i64> keep64(nnz + 1, s), pos(nnz + 1, s);
  keep.zero();
  PMMF_LAUNCH(k_sum_dups, blocks_for(nnz, kThreads), kThreads, 0, s, nnz, keys.get(), v.get(), sums.get(), keep.get(),
              keep_zeros);
  // widen flags to int64 and scan
  PMMF_LAUNCH(k_len64, blocks_for(nnz + 1, kThreads), kThreads, 0, s, nnz, keep.get(), keep64.get());
  exclusive_scan(keep64.get(), pos.get(), nnz + 1, s);
  i64 m = 0;
  PMMF_CUDA(cudaMemcpyAsync(&m, pos.get() + nnz, sizeof(i64), cudaMemcpyDeviceToHost, s));
  PMMF_CUDA(cudaStreamSynchronize(s));
  DBuf<int32_t> col(std::max<i64>(m, 1), s);
  out.row.alloc(std::max<i64>(m, 1), s);
  out.val.alloc(std::max<i64>(m, 1), s);
  PMMF_LAUNCH(k_scatter_kept, blocks_for(nnz, kThreads), kThreads, 0, s, nnz, keys.get(), sums.get(), keep.get(),
              pos.get(), static_cast<uint64_t>(std::max<i64>(N, 1)), col.get(), out.row.get(), out.val.get());
  out.nnz = m;
  out.ptr.alloc(N + 1, s);
  PMMF_LAUNCH(k_ptr_from_cols, blocks_for(m + 1, kThreads), kThreads, 0, s, m, col.get(), N, out.ptr.get());
}

void csc_symmetry(const Csc& a, const Numbering& nb, double* max_asym, double* fro_sq, cudaStream_t s) {
  DBuf<unsigned long long> worst(1, s);
  worst.zero();
  DBuf<double> colfro(std::max<i64>(a.N, 1), s), total(1, s);
  colfro.zero();
  PMMF_LAUNCH(k_symmetry, blocks_for(a.N * 32, kThreads), kThreads, 0, s, a.N, a.ptr.get(), a.row.get(), a.val.get(),
              nb.d_blk.get(), worst.get(), colfro.get());
  size_t tmp = 0;
  PMMF_CUDA(cub::DeviceReduce::Sum(nullptr, tmp, colfro.get(), total.get(), static_cast<int64_t>(std::max<i64>(a.N, 1)), s));
  DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
  PMMF_CUDA(cub::DeviceReduce::Sum(t.get(), tmp, colfro.get(), total.get(), static_cast<int64_t>(std::max<i64>(a.N, 1)), s));
  unsigned long long w = 0;
  PMMF_CUDA(cudaMemcpyAsync(&w, worst.get(), sizeof(w), cudaMemcpyDeviceToHost, s));
  PMMF_CUDA(cudaMemcpyAsync(fro_sq, total.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
  PMMF_CUDA(cudaStreamSynchronize(s));
  double wd;
  std::memcpy(&wd, &w, sizeof(wd));
  *max_asym = wd;
}

void paged_from_csc(Paged& p, Csc&& a, i64 extra_capacity, cudaStream_t s) {
  p.N = a.N;
  p.off.alloc(std::max<i64>(a.N, 1), s);
  p.len.alloc(std::max<i64>(a.N, 1), s);
  PMMF_LAUNCH(k_paged_init, blocks_for(a.N, kThreads), kThreads, 0, s, a.N, a.ptr.get(), p.off.get(), p.len.get());
  p.cap = a.nnz + std::max<i64>(extra_capacity, 1024);
  p.row.alloc(p.cap, s);
  p.val.alloc(p.cap, s);
  if (a.nnz) {
    PMMF_CUDA(cudaMemcpyAsync(p.row.get(), a.row.get(), sizeof(int32_t) * a.nnz, cudaMemcpyDeviceToDevice, s));
    PMMF_CUDA(cudaMemcpyAsync(p.val.get(), a.val.get(), sizeof(double) * a.nnz, cudaMemcpyDeviceToDevice, s));
  }
  p.cursor.alloc(1, s);
  const unsigned long long c0 = static_cast<unsigned long long>(a.nnz);
  PMMF_CUDA(cudaMemcpyAsync(p.cursor.get(), &c0, sizeof(c0), cudaMemcpyHostToDevice, s));
  PMMF_CUDA(cudaStreamSynchronize(s));  // c0 lives on the stack
  a.ptr.release();
  a.row.release();
  a.val.release();
}

void transpose_paged(Csc& out, const Paged& p, cudaStream_t s) {
  const i64 N = p.N;
  DBuf<i64> len64(N + 1, s), pos(N + 1, s);
  PMMF_LAUNCH(k_len64, blocks_for(N + 1, kThreads), kThreads, 0, s, N, p.len.get(), len64.get());
  exclusive_scan(len64.get(), pos.get(), N + 1, s);
  i64 m = 0;
  PMMF_CUDA(cudaMemcpyAsync(&m, pos.get() + N, sizeof(i64), cudaMemcpyDeviceToHost, s));
  PMMF_CUDA(cudaStreamSynchronize(s));
  const int cb = std::max(1, bits_for(std::max<i64>(N - 1, 1)));
  DBuf<uint64_t> keys(std::max<i64>(m, 1), s);
  DBuf<double> vals(std::max<i64>(m, 1), s);
  PMMF_LAUNCH(k_gather_keys, blocks_for(N * 32, kThreads), kThreads, 0, s, N, p.off.get(), p.len.get(), p.row.get(),
              p.val.get(), pos.get(), cb, keys.get(), vals.get());
  // Stable sort on the row bits only: the gather is in (col,row) order, so
  // the result is in (row,col) order.
  sort_pairs(keys, vals, m, cb, 2 * cb, s);
  out.N = N;
  out.nnz = m;
  DBuf<int32_t> major(std::max<i64>(m, 1), s);
  out.row.alloc(std::max<i64>(m, 1), s);
  PMMF_LAUNCH(k_split_keys, blocks_for(m, kThreads), kThreads, 0, s, m, keys.get(), cb, major.get(), out.row.get());
  out.val = std::move(vals);
  out.ptr.alloc(N + 1, s);
  PMMF_LAUNCH(k_ptr_from_cols, blocks_for(m + 1, kThreads), kThreads, 0, s, m, major.get(), N, out.ptr.get());
}

// Row-chunked transpose of pieces: rows [r0, r1) at a time are gathered in
// column order, stable-sorted by row, and handed to `sink` (keys hold
// (row - r0) << cb | column).  Memory: the row histogram plus one chunk.
template <typename Sink>
void transpose_chunks(const std::vector<Piece>& in, i64 N, const uint8_t* keep_row, i64 chunk_nnz,
                      std::vector<i64>& hp, cudaStream_t s, Sink&& sink) {
  const bool tr = trace_enabled();
  auto tl = std::chrono::steady_clock::now();
  double tms[6] = {0, 0, 0, 0, 0, 0};
  auto lap = [&](int k) {
    if (!tr) return;
    PMMF_CUDA(cudaStreamSynchronize(s));
    const auto now = std::chrono::steady_clock::now();
    tms[k] += std::chrono::duration<double, std::milli>(now - tl).count();
    tl = now;
  };
  struct Report {
    bool on;
    double* t;
    ~Report() {
      if (on)
        std::fprintf(stderr, "[pmmf]     transpose: hist %.2f scan %.2f count %.2f gather %.2f sort %.2f sink %.2f ms\n",
                     t[0], t[1], t[2], t[3], t[4], t[5]);
    }
  } report{tr, tms};
  DBuf<int32_t> hist(N + 1, s);
  hist.zero();
  for (const Piece& P : in) {
    const i64 n = P.c1 - P.c0;
    PMMF_LAUNCH(k_row_hist, blocks_for(n * 32, kThreads), kThreads, 0, s, n, P.ptr.get(), P.row.get(), keep_row,
                hist.get());
  }
  lap(0);
  DBuf<i64> h64(N + 1, s), ptr(N + 1, s);
  PMMF_LAUNCH(k_hist_widen, blocks_for(N + 1, kThreads), kThreads, 0, s, N, hist.get(), h64.get());
  exclusive_scan(h64.get(), ptr.get(), N + 1, s);
  hist.release();
  h64.release();
  hp = ptr.to_host(N + 1);
  lap(1);
  const i64 m = hp[N];
  if (m == 0) return;
  chunk_nnz = std::max<i64>(chunk_nnz, 1 << 8);
  DBuf<i64> cnt(N + 1, s), pos(N + 1, s);
  DBuf<uint64_t> keys(std::min(m, chunk_nnz) + 1, s);
  DBuf<double> vals(std::min(m, chunk_nnz) + 1, s);
  const int cb = std::max(1, bits_for(std::max<i64>(N - 1, 1)));
  i64 r0 = 0;
  while (r0 < N) {
    i64 r1 = r0 + 1;
    while (r1 < N && hp[r1 + 1] - hp[r0] <= chunk_nnz) ++r1;
    const i64 cm = hp[r1] - hp[r0];
    if (cm > 0) {
      if (cm > keys.n) {  // a single huge row
        keys.alloc(cm, s);
        vals.alloc(cm, s);
      }
      cnt.zero();
      for (const Piece& P : in) {
        const i64 n = P.c1 - P.c0;
        PMMF_LAUNCH(k_chunk_count, blocks_for(n * 32, kThreads), kThreads, 0, s, n, P.c0, P.ptr.get(), P.row.get(),
                    keep_row, static_cast<int>(r0), static_cast<int>(r1), cnt.get());
      }
      exclusive_scan(cnt.get(), pos.get(), N + 1, s);
      lap(2);
      for (const Piece& P : in) {
        const i64 n = P.c1 - P.c0;
        PMMF_LAUNCH(k_chunk_gather, blocks_for(n * 32, kThreads), kThreads, 0, s, n, P.c0, P.ptr.get(), P.row.get(),
                    P.val.get(), keep_row, static_cast<int>(r0), static_cast<int>(r1), pos.get(), cb, keys.get(),
                    vals.get());
      }
      lap(3);
      const int rb = std::max(1, bits_for(std::max<i64>(r1 - r0 - 1, 1)));
      DBuf<uint64_t> k2(cm, s);
      DBuf<double> v2(cm, s);
      cub::DoubleBuffer<uint64_t> kb(keys.get(), k2.get());
      cub::DoubleBuffer<double> vb(vals.get(), v2.get());
      size_t tmp = 0;
      PMMF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, static_cast<int64_t>(cm), cb, cb + rb, s));
      DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
      PMMF_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, kb, vb, static_cast<int64_t>(cm), cb, cb + rb, s));
      lap(4);
      sink(r0, r1, cm, cb, kb.Current(), vb.Current(), ptr.get());
      lap(5);
    }
    r0 = r1;
  }
}

void transpose_pieces(Csc& out, const std::vector<Piece>& in, i64 N, const uint8_t* keep_row, i64 chunk_nnz,
                      cudaStream_t s) {
  out.N = N;
  std::vector<i64> hp;
  // sizes first (the histogram pass of transpose_chunks), then the chunks
  out.ptr.alloc(N + 1, s);
  bool allocated = false;
  transpose_chunks(in, N, keep_row, chunk_nnz, hp, s,
                   [&](i64 r0, i64, i64 cm, int cb, const uint64_t* keys, const double* vals, const i64*) {
                     if (!allocated) {
                       out.row.alloc(std::max<i64>(hp[N], 1), s);
                       out.val.alloc(std::max<i64>(hp[N], 1), s);
                       allocated = true;
                     }
                     PMMF_LAUNCH(k_chunk_emit, blocks_for(cm, kThreads), kThreads, 0, s, cm, keys, vals, cb,
                                 out.row.get() + hp[r0], out.val.get() + hp[r0]);
                   });
  out.nnz = hp.empty() ? 0 : hp[N];
  if (!allocated) {
    out.row.alloc(std::max<i64>(out.nnz, 1), s);
    out.val.alloc(std::max<i64>(out.nnz, 1), s);
  }
  if (!hp.empty()) out.ptr.upload(hp);
}


void reblock(Csc& out, const Csc& a, const DBuf<int32_t>& map, const DBuf<int32_t>& new2old, i64 n_new,
             cudaStream_t s) {
  const auto t_start = std::chrono::steady_clock::now();
  DBuf<i64> cnt(n_new + 1, s), nptr(n_new + 1, s);
  PMMF_LAUNCH(k_reblock_count, blocks_for((n_new + 1) * 32, kThreads), kThreads, 0, s, n_new, new2old.get(),
              a.ptr.get(), a.row.get(), map.get(), cnt.get());
  exclusive_scan(cnt.get(), nptr.get(), n_new + 1, s);
  i64 m = 0;
  PMMF_CUDA(cudaMemcpyAsync(&m, nptr.get() + n_new, sizeof(i64), cudaMemcpyDeviceToHost, s));
  PMMF_CUDA(cudaStreamSynchronize(s));
  DBuf<int32_t> r1(std::max<i64>(m, 1), s);
  DBuf<double> v1(std::max<i64>(m, 1), s);
  PMMF_LAUNCH(k_reblock_fill, blocks_for(n_new * 32, kThreads), kThreads, 0, s, n_new, new2old.get(), a.ptr.get(),
              a.row.get(), a.val.get(), map.get(), nptr.get(), r1.get(), v1.get());
  double t_fill = 0.0;
  if (trace_enabled()) {
    PMMF_CUDA(cudaStreamSynchronize(s));
    t_fill = ms_since_tp(t_start);
  }
  const auto t_sort0 = std::chrono::steady_clock::now();
  out.N = n_new;
  out.nnz = m;
  out.row.alloc(std::max<i64>(m, 1), s);
  out.val.alloc(std::max<i64>(m, 1), s);
  if (m > 0 && n_new > 0) {
    size_t tmp = 0;
    PMMF_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, tmp, r1.get(), out.row.get(), v1.get(), out.val.get(),
                                                  static_cast<int64_t>(m), static_cast<int64_t>(n_new), nptr.get(),
                                                  nptr.get() + 1, s));
    DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
    PMMF_CUDA(cub::DeviceSegmentedSort::SortPairs(t.get(), tmp, r1.get(), out.row.get(), v1.get(), out.val.get(),
                                                  static_cast<int64_t>(m), static_cast<int64_t>(n_new), nptr.get(),
                                                  nptr.get() + 1, s));
  }
  out.ptr = std::move(nptr);
  if (trace_enabled()) {
    PMMF_CUDA(cudaStreamSynchronize(s));
    std::fprintf(stderr, "[pmmf]   reblock: count+fill %.2f ms, sort %.2f ms\n", t_fill, ms_since_tp(t_sort0));
  }
}

}  // namespace pmmf_b200
