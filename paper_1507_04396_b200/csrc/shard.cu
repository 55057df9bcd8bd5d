// shard.cu — multi-GPU plumbing of the sharded stage loop (shard.cuh):
// the cluster split, the in-place segment broadcasts over NCCL and the
// gather of the per-rank column slabs; plus the communicator half of the
// C-ABI.  The reference runs the independent clusters of a stage on a
// fork-join thread pool (parallel.hpp:25-71, factorizer.hpp:494-504 and
// :513); here they run on W GPUs.
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

}  // namespace

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

void csc_gather_slabs(Csc& out, std::vector<Csc>& parts, const std::vector<i64>& col_seg, i64 N, const Comm& c,
                      cudaStream_t s) {
  const std::vector<int> mine = c.local_ranks();
  const int W = c.size;
  // slab sizes of every rank
  std::vector<i64> nnz(static_cast<size_t>(W), 0);
  for (size_t i = 0; i < mine.size(); ++i) nnz[mine[i]] = parts[i].nnz;
  if (c.multi_process()) {
    DBuf<i64> d(W, s);
    d.upload(nnz);
    std::vector<i64> seg(static_cast<size_t>(W) + 1);
    for (int r = 0; r <= W; ++r) seg[r] = r;
    bcast_segments(d.get(), sizeof(i64), seg, c, s);
    nnz = d.to_host(W);
  }
  std::vector<i64> base(static_cast<size_t>(W) + 1, 0);
  for (int r = 0; r < W; ++r) base[r + 1] = base[r] + nnz[r];
  const i64 total = base[W];
  out = Csc();
  out.N = N;
  out.nnz = total;
  out.ptr.alloc(N + 1, s);
  out.row.alloc(std::max<i64>(total, 1), s);
  out.val.alloc(std::max<i64>(total, 1), s);
  for (size_t i = 0; i < mine.size(); ++i) {
    const int r = mine[i];
    Csc& P = parts[i];
    const i64 c0 = col_seg[r], c1 = col_seg[r + 1];
    // the slab's entries are contiguous: columns outside [c0, c1) are empty
    if (c1 > c0) {
      i64 p0 = 0;
      PMMF_CUDA(cudaMemcpyAsync(&p0, P.ptr.get() + c0, sizeof(i64), cudaMemcpyDeviceToHost, s));
      PMMF_CUDA(cudaStreamSynchronize(s));
      if (p0 != 0) fail(PMMF_INTERNAL, "csc_gather_slabs: slab has entries before its column range");
      PMMF_LAUNCH(k_ptr_shift, blocks_for(c1 - c0, kThreads), kThreads, 0, s, c1 - c0, P.ptr.get() + c0, i64{0},
                  base[r], out.ptr.get() + c0);
    }
    if (nnz[r] > 0) {
      PMMF_CUDA(cudaMemcpyAsync(out.row.get() + base[r], P.row.get(), sizeof(int32_t) * nnz[r],
                                cudaMemcpyDeviceToDevice, s));
      PMMF_CUDA(cudaMemcpyAsync(out.val.get() + base[r], P.val.get(), sizeof(double) * nnz[r],
                                cudaMemcpyDeviceToDevice, s));
    }
    P = Csc();
  }
  PMMF_CUDA(cudaMemcpyAsync(out.ptr.get() + N, &total, sizeof(i64), cudaMemcpyHostToDevice, s));
  bcast_segments(out.ptr.get(), sizeof(i64), col_seg, c, s);
  bcast_segments(out.row.get(), sizeof(int32_t), base, c, s);
  bcast_segments(out.val.get(), sizeof(double), base, c, s);
  PMMF_CUDA(cudaStreamSynchronize(s));  // `total` is a host stack value
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
