// common.cuh — error model, device buffers and launch accounting shared by
// every translation unit of libpmmf_b200.so.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <map>
#include <mutex>
#include <chrono>
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

// Diagnostic (PMMF_B200_SLOWCALL=<ms>): reports any instrumented host call
// (allocation, copy, launch, memset) that blocks longer than the threshold --
// host-side stalls inside the launch-bound late stages show up here.
inline double slowcall_ms() {
  static const double v = [] {
    const char* e = std::getenv("PMMF_B200_SLOWCALL");
    return e ? std::atof(e) : 0.0;
  }();
  return v;
}
struct SlowCall {
  const char* what;
  size_t arg;
  std::chrono::steady_clock::time_point t0;
  bool on;
  explicit SlowCall(const char* w, size_t a = 0) : what(w), arg(a), on(slowcall_ms() > 0.0) {
    if (on) t0 = std::chrono::steady_clock::now();
  }
  ~SlowCall() {
    if (!on) return;
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (ms > slowcall_ms()) std::fprintf(stderr, "[pmmf] slow call: %s (%zu) %.2f ms\n", what, arg, ms);
  }
};

// Every kernel launch in csrc/ goes through PMMF_LAUNCH so the library can
// report how many of its own kernels ran (bench.py "gpu_launches").
std::atomic<int64_t>& launch_counter();
#define PMMF_LAUNCH(kernel, grid, block, smem, stream, ...)                  \
  do {                                                                       \
    if ((grid) > 0) {                                                        \
      ::pmmf_b200::SlowCall slow_(#kernel);                                  \
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

// Large blocks (>= kBigBytes) are cached whole instead of going back to the
// stream-ordered pool: a fresh mapping of tens of GB costs ~80 ms per GB
// (measured), and the pool, fragmented by the stage's mixed lifetimes, would
// otherwise re-map the row-pass arenas, Gram tiles and sort buffers every
// stage.  A cached block serves a request of at most its size and at least
// 2/3 of it; it is reused on any stream after the event recorded at its
// release.  On allocation failure the cache is emptied and the pool trimmed.
constexpr size_t kBigBytes = size_t{32} << 20;

struct BigCache {
  struct Blk {
    void* p;
    size_t bytes;
    int dev;
    cudaEvent_t ready;
  };
  std::mutex mu;
  std::vector<Blk> blocks;
  size_t cached = 0;
  static BigCache& get() {
    static BigCache c;
    return c;
  }
  // Best fit among cached blocks; nullptr if none qualifies.  Requests
  // below 1 GB are power-of-two size classes (pool_alloc) and take a block
  // of their class or the next; larger ones a block within 1.5x.
  void* take(size_t bytes, int dev, cudaStream_t st, size_t* got) {
    std::lock_guard<std::mutex> g(mu);
    size_t best = blocks.size();
    const size_t lim = bytes < (size_t{1} << 30) ? 2 * bytes : bytes + bytes / 2;
    for (size_t i = 0; i < blocks.size(); ++i) {
      const Blk& b = blocks[i];
      if (b.dev != dev || b.bytes < bytes || b.bytes > lim) continue;
      if (best == blocks.size() || b.bytes < blocks[best].bytes) best = i;
    }
    if (best == blocks.size()) return nullptr;
    Blk b = blocks[best];
    blocks.erase(blocks.begin() + static_cast<std::ptrdiff_t>(best));
    cached -= b.bytes;
    cudaStreamWaitEvent(st, b.ready, 0);
    cudaEventDestroy(b.ready);
    *got = b.bytes;
    return b.p;
  }
  void give(void* p, size_t bytes, int dev, cudaStream_t st) {
    cudaEvent_t ev = nullptr;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (cudaEventRecord(ev, st) != cudaSuccess)
      std::fprintf(stderr, "[pmmf] cache: event record failed on stream %p: %s\n", static_cast<void*>(st),
                   cudaGetErrorString(cudaGetLastError()));
    std::lock_guard<std::mutex> g(mu);
    blocks.push_back({p, bytes, dev, ev});
    cached += bytes;
  }
  // Returns every cached block of `dev` to the pool (after its last use).
  void drain(int dev, cudaStream_t st) {
    std::lock_guard<std::mutex> g(mu);
    std::vector<Blk> keep;
    for (Blk& b : blocks) {
      if (b.dev != dev) {
        keep.push_back(b);
        continue;
      }
      cudaEventSynchronize(b.ready);
      cudaEventDestroy(b.ready);
      if (trace_enabled() || std::getenv("PMMF_B200_ALLOC_CHECK"))
        std::fprintf(stderr, "[pmmf]   cache drain frees %p+%zu\n", b.p, b.bytes);
      cudaFreeAsync(b.p, st);
      cached -= b.bytes;
    }
    blocks.swap(keep);
  }
  size_t cached_bytes() {
    std::lock_guard<std::mutex> g(mu);
    return cached;
  }
};

// Debug registry of live large blocks (PMMF_B200_ALLOC_CHECK): reports a
// block handed out twice or released while not live.
struct AllocCheck {
  std::mutex mu;
  std::map<void*, size_t> live;
  static AllocCheck& get() {
    static AllocCheck a;
    return a;
  }
  static bool on() {
    static const bool f = std::getenv("PMMF_B200_ALLOC_CHECK") != nullptr;
    return f;
  }
  static bool verbose() {
    static const bool f = std::getenv("PMMF_B200_ALLOC_CHECK") && std::getenv("PMMF_B200_ALLOC_CHECK")[0] == '2';
    return f;
  }
  void add(void* p, size_t b, const char* how) {
    std::lock_guard<std::mutex> g(mu);
    if (verbose()) std::fprintf(stderr, "[ac] +%s %p %zu\n", how, p, b);
    auto it = live.lower_bound(p);
    if (it != live.end() && static_cast<char*>(it->first) < static_cast<char*>(p) + b)
      std::fprintf(stderr, "[pmmf] alloc-check: %s %p+%zu overlaps live %p+%zu\n", how, p, b, it->first, it->second);
    if (it != live.begin()) {
      --it;
      if (static_cast<char*>(it->first) + it->second > static_cast<char*>(p))
        std::fprintf(stderr, "[pmmf] alloc-check: %s %p+%zu overlaps live %p+%zu\n", how, p, b, it->first, it->second);
    }
    live[p] = b;
  }
  void remove(void* p, size_t b) {
    std::lock_guard<std::mutex> g(mu);
    if (verbose()) std::fprintf(stderr, "[ac] -free %p %zu\n", p, b);
    auto it = live.find(p);
    if (it == live.end())
      std::fprintf(stderr, "[pmmf] alloc-check: release of non-live %p+%zu\n", p, b);
    else
      live.erase(it);
  }
};

// Grow-only pinned host staging (device->host copies of the rotation records
// run at full PCIe/C2C speed; pinned memory is never freed, so no implicit
// device synchronisation).  A slot is held under its lock while in use.
struct PinnedSlot {
  std::mutex mu;
  void* p = nullptr;
  size_t bytes = 0;
  void* reserve(size_t n) {  // caller holds mu
    if (n > bytes) {
      void* q = nullptr;
      if (cudaHostAlloc(&q, n, cudaHostAllocDefault) != cudaSuccess) {
        (void)cudaGetLastError();
        return nullptr;
      }
      p = q;  // the previous block is kept (never freed): no implicit sync
      bytes = n;
    }
    return p;
  }
  static PinnedSlot& get(int i) {
    static PinnedSlot slots[4];
    return slots[i & 3];
  }
};

// Reusable timing events for the profiled passes (creating and destroying
// two events per dependency level would itself cost ~10 us a level).
struct EventPool {
  std::mutex mu;
  std::vector<cudaEvent_t> free_ev;
  static EventPool& get() {
    static EventPool p;
    return p;
  }
  cudaEvent_t take() {
    {
      std::lock_guard<std::mutex> g(mu);
      if (!free_ev.empty()) {
        cudaEvent_t e = free_ev.back();
        free_ev.pop_back();
        return e;
      }
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
  void give(cudaEvent_t e) {
    std::lock_guard<std::mutex> g(mu);
    free_ev.push_back(e);
  }
};

// The library's own stream-ordered memory pool per device (not the device's
// default pool, whose settings belong to the process: torch and other
// cudaMallocAsync users).  Freed blocks stay mapped (release threshold =
// max): re-mapping tens of GB per stage costs seconds; pool_alloc trims it
// when fragmentation alone fails a request, pmmf_b200_cached_bytes(dev, 1)
// hands everything back.
inline cudaMemPool_t lib_pool(int dev) {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  std::lock_guard<std::mutex> g(mu);
  auto it = pools.find(dev);
  if (it != pools.end()) return it->second;
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.handleTypes = cudaMemHandleTypeNone;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool = nullptr;
  PMMF_CUDA(cudaMemPoolCreate(&pool, &props));
  uint64_t thr = ~uint64_t{0};
  if (const char* e = std::getenv("PMMF_B200_POOL_KEEP_GB")) thr = static_cast<uint64_t>(std::atof(e) * 1073741824.0);
  PMMF_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  pools[dev] = pool;
  return pool;
}

// Device memory a new allocation can still get: free memory, the pool's
// reserved-but-unused blocks and the cached large blocks.
inline i64 available_bytes() {
  size_t f = 0, t = 0;
  PMMF_CUDA(cudaMemGetInfo(&f, &t));
  int dev = 0;
  PMMF_CUDA(cudaGetDevice(&dev));
  cudaMemPool_t pool = lib_pool(dev);
  uint64_t reserved = 0, used = 0;
  PMMF_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
  PMMF_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
  return static_cast<i64>(f) + static_cast<i64>(reserved - used) + static_cast<i64>(BigCache::get().cached_bytes());
}

// Bytes of large blocks that missed the cache (fresh pool allocations):
// a steady-state factorization should add none (PMMF_B200_TRACE reports it).
inline std::atomic<uint64_t>& fresh_big_bytes() {
  static std::atomic<uint64_t> b{0};
  return b;
}

// Stream-ordered allocation.  Large requests are rounded up (64 MB above
// 1 GB, 4 MB below) and
// served from the block cache when possible.  A failed request drains the
// cache, trims the pool and is retried once.  *bytes is updated to the size
// actually held.
inline void pool_alloc(void** p, size_t* bytes, cudaStream_t st) {
  SlowCall slow_("pool_alloc", *bytes);
  int dev = 0;
  PMMF_CUDA(cudaGetDevice(&dev));
  if (*bytes >= kBigBytes) {
    // mid-size blocks (32 MB .. 1 GB) in power-of-two classes: the sizes a
    // stage asks for vary from step to step and stage to stage, and a class
    // that misses the cache maps fresh memory (~80 ms per GB, more when the
    // device is nearly full); the largest blocks keep 64 MB granularity
    if (*bytes < (size_t{1} << 30)) {
      size_t c = kBigBytes;
      while (c < *bytes) c <<= 1;
      *bytes = c;
    } else {
      const size_t g = size_t{64} << 20;
      *bytes = (*bytes + g - 1) / g * g;
    }
    size_t got = 0;
    if (void* q = BigCache::get().take(*bytes, dev, st, &got)) {
      *p = q;
      *bytes = got;
      if (AllocCheck::on()) AllocCheck::get().add(q, got, "cache");
      return;
    }
  }
  if (*bytes >= kBigBytes) fresh_big_bytes().fetch_add(*bytes, std::memory_order_relaxed);  // cache missed
  const bool timed = *bytes >= (size_t{64} << 20) && trace_enabled();
  std::chrono::steady_clock::time_point t0;
  if (timed) {
    cudaStreamSynchronize(st);
    t0 = std::chrono::steady_clock::now();
  }
  cudaError_t e = cudaMallocFromPoolAsync(p, *bytes, lib_pool(dev), st);
  if (e == cudaErrorMemoryAllocation) {
    (void)cudaGetLastError();
    PMMF_CUDA(cudaStreamSynchronize(st));
    BigCache::get().drain(dev, st);
    PMMF_CUDA(cudaStreamSynchronize(st));
    PMMF_CUDA(cudaMemPoolTrimTo(lib_pool(dev), 0));
    if (trace_enabled()) std::fprintf(stderr, "[pmmf]   pool trimmed for a %zu MB request\n", *bytes >> 20);
    e = cudaMallocFromPoolAsync(p, *bytes, lib_pool(dev), st);
  }
  PMMF_CUDA(e);
  if (AllocCheck::on()) AllocCheck::get().add(*p, *bytes, "malloc");
  if (timed) {
    cudaStreamSynchronize(st);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (ms > 2.0) std::fprintf(stderr, "[pmmf]   slow alloc: %zu MB in %.1f ms\n", *bytes >> 20, ms);
  }
}
inline void pool_free(void* p, size_t bytes, cudaStream_t st) {
  SlowCall slow_("pool_free", bytes);
  if (AllocCheck::on()) AllocCheck::get().remove(p, bytes);
  if (bytes >= kBigBytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    BigCache::get().give(p, bytes, dev, st);
  } else {
    cudaFreeAsync(p, st);
  }
}

// Stream-ordered device buffer (from the library's pool, lib_pool).
template <typename T>
struct DBuf {
  T* p = nullptr;
  i64 n = 0;
  size_t held = 0;  // bytes held (>= n * sizeof(T))
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
      held = o.held;
      s = o.s;
      o.p = nullptr;
      o.n = 0;
      o.held = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(i64 count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count > 0) {
      held = sizeof(T) * static_cast<size_t>(count);
      pool_alloc(reinterpret_cast<void**>(&p), &held, st);
    }
  }
  void release() noexcept {
    if (p) pool_free(p, held, s);
    p = nullptr;
    n = 0;
    held = 0;
  }
  T* get() const { return p; }
  void zero(const char* file = __builtin_FILE(), int line = __builtin_LINE()) const {
    if (n) {
      const cudaError_t e = cudaMemsetAsync(p, 0, sizeof(T) * static_cast<size_t>(n), s);
      if (e != cudaSuccess) {
        cudaPointerAttributes at{};
        const cudaError_t e2 = cudaPointerGetAttributes(&at, p);
        std::fprintf(stderr, "[pmmf] memset failed at %s:%d: p=%p bytes=%zu held=%zu stream=%p attr=%d type=%d dev=%d\n",
                     file, line, static_cast<void*>(p), sizeof(T) * static_cast<size_t>(n), held, static_cast<void*>(s),
                     static_cast<int>(e2), static_cast<int>(at.type), at.device);
      }
      PMMF_CUDA(e);
    }
  }
  void fill_bytes(int v) const {
    if (n) PMMF_CUDA(cudaMemsetAsync(p, v, sizeof(T) * static_cast<size_t>(n), s));
  }
  void upload(const T* h, i64 count) const {
    SlowCall slow_("upload", sizeof(T) * static_cast<size_t>(count));
    if (count) PMMF_CUDA(cudaMemcpyAsync(p, h, sizeof(T) * static_cast<size_t>(count), cudaMemcpyHostToDevice, s));
  }
  void upload(const std::vector<T>& h) const { upload(h.data(), static_cast<i64>(h.size())); }
  void download(T* h, i64 count) const {
    SlowCall slow_("download", sizeof(T) * static_cast<size_t>(count));
    if (count) PMMF_CUDA(cudaMemcpyAsync(h, p, sizeof(T) * static_cast<size_t>(count), cudaMemcpyDeviceToHost, s));
  }
  std::vector<T> to_host(i64 count) const {
    SlowCall slow_("to_host", sizeof(T) * static_cast<size_t>(count));
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
