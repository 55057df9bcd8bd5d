// common.cuh — error model, device buffers and launch accounting shared by
// every translation unit of libpmmf_b200.so.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/pmmf_b200.h"

namespace pmmf_b200 {

using i64 = int64_t;

// Mirrors the reference's exception taxonomy (types.hpp:24-32); the C-ABI
// turns it into a pmmf_b200_status.
struct Error {
  int code;
  std::string msg;
};
[[noreturn]] inline void fail(int code, const std::string& m) { throw Error{code, m}; }

#define PMMF_CUDA(call)                                                                     \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      ::pmmf_b200::fail(PMMF_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_) +     \
                                       " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"); \
  } while (0)

// Every kernel launch in csrc/ goes through PMMF_LAUNCH so the library can
// report how many of its own kernels ran (bench.py "gpu_launches").
std::atomic<int64_t>& launch_counter();
#define PMMF_LAUNCH(kernel, grid, block, smem, stream, ...)                  \
  do {                                                                       \
    if ((grid) > 0) {                                                        \
      kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);            \
      ::pmmf_b200::launch_counter().fetch_add(1, std::memory_order_relaxed); \
      PMMF_CUDA(cudaGetLastError());                                         \
    }                                                                        \
  } while (0)

// Live per-kernel accounting for bench.py's roofline: when enabled, the
// instrumented launch sites bracket their kernel with CUDA events on the
// launching stream and add the algorithmic bytes they moved.
struct ProfStat {
  int64_t launches = 0;
  double ms = 0.0;
  double bytes = 0.0;
};
bool prof_enabled();
void prof_set(bool on);
bool prof_get(const char* name, ProfStat* out);
void prof_add(const char* name, double ms, double bytes);
void prof_add_n(const char* name, int64_t launches, double ms, double bytes);
struct ProfScope {
  const char* name;
  cudaStream_t s;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  ProfScope(const char* n, cudaStream_t st) : name(n), s(st) {
    if (prof_enabled()) {
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, s);
    }
  }
  // call after the launch; bytes known by then or passed later via finish
  void finish(double bytes) {
    if (!e0) return;
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    prof_add(name, ms, bytes);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    e0 = e1 = nullptr;
  }
  ~ProfScope() {
    if (e0) {
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
  }
};

// PMMF_B200_TRACE=1 prints per-stage diagnostics to stderr.
inline bool trace_enabled() {
  const char* e = std::getenv("PMMF_B200_TRACE");  // read per call: cheap, and togglable
  return e && *e && *e != '0';
}

// Device memory a new allocation can still get: free memory plus the pool's
// reserved-but-unused blocks.
inline i64 available_bytes() {
  size_t f = 0, t = 0;
  PMMF_CUDA(cudaMemGetInfo(&f, &t));
  int dev = 0;
  PMMF_CUDA(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  PMMF_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t reserved = 0, used = 0;
  PMMF_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
  PMMF_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
  return static_cast<i64>(f) + static_cast<i64>(reserved - used);
}

// Stream-ordered allocation from the device pool.  The pool keeps freed
// blocks mapped (mapping is the expensive part), so a large request can fail
// on fragmentation alone: then the stream is drained, the pool trimmed back to
// what is in use, and the request retried once.
inline void pool_alloc(void** p, size_t bytes, cudaStream_t st) {
  cudaError_t e = cudaMallocAsync(p, bytes, st);
  if (e == cudaErrorMemoryAllocation) {
    (void)cudaGetLastError();
    PMMF_CUDA(cudaStreamSynchronize(st));
    int dev = 0;
    PMMF_CUDA(cudaGetDevice(&dev));
    cudaMemPool_t pool;
    PMMF_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    PMMF_CUDA(cudaMemPoolTrimTo(pool, 0));
    if (trace_enabled()) std::fprintf(stderr, "[pmmf]   pool trimmed for a %zu MB request\n", bytes >> 20);
    e = cudaMallocAsync(p, bytes, st);
  }
  PMMF_CUDA(e);
}

// Stream-ordered device buffer (cudaMallocAsync from the device pool).
template <typename T>
struct DBuf {
  T* p = nullptr;
  i64 n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(i64 count, cudaStream_t st) { alloc(count, st); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept { *this = std::move(o); }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      s = o.s;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(i64 count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count > 0) pool_alloc(reinterpret_cast<void**>(&p), sizeof(T) * static_cast<size_t>(count), st);
  }
  void release() noexcept {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  T* get() const { return p; }
  void zero() const {
    if (n) PMMF_CUDA(cudaMemsetAsync(p, 0, sizeof(T) * static_cast<size_t>(n), s));
  }
  void fill_bytes(int v) const {
    if (n) PMMF_CUDA(cudaMemsetAsync(p, v, sizeof(T) * static_cast<size_t>(n), s));
  }
  void upload(const T* h, i64 count) const {
    if (count) PMMF_CUDA(cudaMemcpyAsync(p, h, sizeof(T) * static_cast<size_t>(count), cudaMemcpyHostToDevice, s));
  }
  void upload(const std::vector<T>& h) const { upload(h.data(), static_cast<i64>(h.size())); }
  void download(T* h, i64 count) const {
    if (count) PMMF_CUDA(cudaMemcpyAsync(h, p, sizeof(T) * static_cast<size_t>(count), cudaMemcpyDeviceToHost, s));
  }
  std::vector<T> to_host(i64 count) const {
    std::vector<T> h(static_cast<size_t>(count));
    download(h.data(), count);
    PMMF_CUDA(cudaStreamSynchronize(s));
    return h;
  }
};

inline unsigned blocks_for(i64 n, int threads) {
  return static_cast<unsigned>((n + threads - 1) / threads);
}

inline int bits_for(i64 x) {  // smallest b with 2^b > x (x >= 0)
  int b = 0;
  while (b < 63 && (i64{1} << b) <= x) ++b;
  return b;
}

// Exact fp64 arithmetic without contraction: every product and sum rounds
// separately, as the reference's x86-64 -O2 build does.
#ifdef __CUDACC__
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
#endif

}  // namespace pmmf_b200
