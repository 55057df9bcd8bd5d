// abi.cu — the C-ABI of include/pmmf_b200.h: status mapping, the
// factorization entry point and the MmfFactorization accessors.
#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <string>

#include "result.cuh"
#include "rotation.cuh"
#include "shard.cuh"

using namespace pmmf_b200;

namespace {

void set_err(char* err, size_t n, const std::string& m) {
  if (!err || !n) return;
  const size_t k = std::min(n - 1, m.size());
  std::memcpy(err, m.data(), k);
  err[k] = '\0';
}

}  // namespace

namespace pmmf_b200 {
namespace {
std::mutex& prof_mu() {
  static std::mutex m;
  return m;
}
std::map<std::string, ProfStat>& prof_map() {
  static std::map<std::string, ProfStat> m;
  return m;
}
std::atomic<bool>& prof_flag() {
  static std::atomic<bool> f{false};
  return f;
}
}  // namespace
bool prof_enabled() { return prof_flag().load(std::memory_order_relaxed); }
void prof_set(bool on) {
  std::lock_guard<std::mutex> g(prof_mu());
  prof_flag() = on;
  prof_map().clear();
}
bool prof_get(const char* name, ProfStat* out) {
  std::lock_guard<std::mutex> g(prof_mu());
  auto it = prof_map().find(name);
  if (it == prof_map().end()) return false;
  *out = it->second;
  return true;
}
void prof_add(const char* name, double ms, double bytes) {
  std::lock_guard<std::mutex> g(prof_mu());
  ProfStat& s = prof_map()[name];
  ++s.launches;
  s.ms += ms;
  s.bytes += bytes;
}
void prof_add_n(const char* name, int64_t launches, double ms, double bytes) {
  std::lock_guard<std::mutex> g(prof_mu());
  ProfStat& s = prof_map()[name];
  s.launches += launches;
  s.ms += ms;
  s.bytes += bytes;
}
int guarded_call(char* err, size_t errlen, void (*fn)(void*), void* ctx) {
  try {
    fn(ctx);
    return PMMF_OK;
  } catch (const Error& e) {
    set_err(err, errlen, e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_err(err, errlen, "host allocation failed");
    return PMMF_INTERNAL;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return PMMF_INTERNAL;
  }
}
}  // namespace pmmf_b200

template <typename F>
static int guarded(char* err, size_t errlen, F&& f) {
  return guarded_call(err, errlen, [](void* c) { (*static_cast<F*>(c))(); }, &f);
}

extern "C" {

int pmmf_b200_factorize(const pmmf_b200_coo* a, const pmmf_b200_params* p, void** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!a || !p || !out) fail(PMMF_INVALID_ARGUMENT, "pmmf_b200_factorize: null argument");
    *out = factorize_device(a, *p).release();
  });
}

int pmmf_b200_factorize_sharded(const pmmf_b200_coo* a, const pmmf_b200_params* p, void* comm, void** out,
                                char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!a || !p || !out || !comm) fail(PMMF_INVALID_ARGUMENT, "pmmf_b200_factorize_sharded: null argument");
    *out = factorize_device(a, *p, static_cast<const Comm*>(comm)).release();
  });
}

int pmmf_b200_result_save(void* h, const char* path, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!h || !path) fail(PMMF_INVALID_ARGUMENT, "pmmf_b200_result_save: null argument");
    save_factorization(*static_cast<Result*>(h), path);
  });
}

int pmmf_b200_result_load(const char* path, void** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!path || !out) fail(PMMF_INVALID_ARGUMENT, "pmmf_b200_result_load: null argument");
    *out = load_factorization(path).release();
  });
}

int pmmf_b200_result_params(void* h, pmmf_b200_params* out) {
  if (!h || !out) return PMMF_INVALID_ARGUMENT;
  *out = static_cast<Result*>(h)->params;
  return PMMF_OK;
}

int pmmf_b200_result_create(int64_t n, const pmmf_b200_params* p, double residual_sq, void** out, char* err,
                            size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!p || !out) fail(PMMF_INVALID_ARGUMENT, "pmmf_b200_result_create: null argument");
    if (n < 0) fail(PMMF_DATA, "factorization: negative n");
    if (p->k < 2 || p->k > kMaxK) fail(PMMF_DATA, "factorization: params.k outside [2, 8]");
    auto r = std::make_unique<Result>();
    r->n = n;
    r->k = p->k;
    r->params = *p;
    r->residual_sq = residual_sq;
    r->trivial = true;
    *out = r.release();
  });
}

int pmmf_b200_result_add_stage(void* h, int64_t n_clusters, const int64_t* offs, const int64_t* mem, int64_t nr,
                               const int64_t* ri, const double* rq, int64_t ne, const int64_t* ei, const double* ed,
                               const double* em, int64_t nb, const int64_t* by, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!h || !offs || n_clusters < 0 || nr < 0 || ne < 0 || nb < 0)
      fail(PMMF_INVALID_ARGUMENT, "pmmf_b200_result_add_stage: bad argument");
    auto* r = static_cast<Result*>(h);
    const int64_t k = r->k;
    const int64_t np = offs[n_clusters];
    if ((np && !mem) || (nr && (!ri || !rq)) || (ne && (!ei || !ed || !em)) || (nb && !by))
      fail(PMMF_INVALID_ARGUMENT, "pmmf_b200_result_add_stage: null array");
    Result::Stage st;
    st.off.assign(offs, offs + n_clusters + 1);
    if (np < 0) fail(PMMF_DATA, "factorization: inconsistent partition offsets");
    st.members.assign(mem, mem + np);
    st.rot_idx.assign(ri, ri + nr * k);
    st.rot_q.assign(rq, rq + nr * k * k);
    st.elim_idx.assign(ei, ei + ne);
    st.elim_diag.assign(ed, ed + ne);
    st.elim_mass.assign(em, em + ne);
    st.bypassed.assign(by, by + nb);
    r->stages.push_back(std::move(st));
    r->trivial = false;
  });
}

int pmmf_b200_result_set_core(void* h, int64_t g, const int64_t* ci, const double* core, int64_t nd,
                              const int64_t* di, const double* dv, const int64_t* hist, int64_t nh, char* err,
                              size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!h || g < 0 || nd < 0 || nh < 0 || (g && (!ci || !core)) || (nd && (!di || !dv)) || (nh && !hist))
      fail(PMMF_INVALID_ARGUMENT, "pmmf_b200_result_set_core: bad argument");
    auto* r = static_cast<Result*>(h);
    r->core_idx.assign(ci, ci + g);
    r->core.assign(core, core + g * g);
    r->diag.clear();
    for (int64_t i = 0; i < nd; ++i) r->diag.emplace_back(di[i], dv[i]);
    r->hist.assign(hist, hist + nh);
    validate_result(*r);
  });
}

int pmmf_b200_result_summary(void* h, pmmf_b200_summary* o) {
  if (!h || !o) return PMMF_INVALID_ARGUMENT;
  auto* r = static_cast<Result*>(h);
  o->n = r->n;
  o->n_stages = static_cast<int64_t>(r->stages.size());
  o->k = r->k;
  o->core_size = static_cast<int64_t>(r->core_idx.size());
  o->n_diagonal = static_cast<int64_t>(r->diag.size());
  o->trivial = r->trivial;
  o->residual_sq = r->residual_sq;
  return PMMF_OK;
}

int pmmf_b200_result_active_history(void* h, int64_t* o) {
  if (!h || (!o && !static_cast<Result*>(h)->hist.empty())) return PMMF_INVALID_ARGUMENT;
  auto* r = static_cast<Result*>(h);
  std::copy(r->hist.begin(), r->hist.end(), o);
  return PMMF_OK;
}

int pmmf_b200_result_stage_sizes(void* h, int64_t s, pmmf_b200_stage_sizes* o) {
  if (!h || !o) return PMMF_INVALID_ARGUMENT;
  auto* r = static_cast<Result*>(h);
  if (s < 0 || s >= static_cast<int64_t>(r->stages.size())) return PMMF_OUT_OF_RANGE;
  const auto& st = r->stages[s];
  o->n_clusters = static_cast<int64_t>(st.off.size()) - 1;
  o->partition_size = static_cast<int64_t>(st.members.size());
  o->n_rotations = static_cast<int64_t>(st.rot_idx.size()) / r->k;
  o->n_eliminated = static_cast<int64_t>(st.elim_idx.size());
  o->n_bypassed = static_cast<int64_t>(st.bypassed.size());
  return PMMF_OK;
}

int pmmf_b200_result_stage(void* h, int64_t s, int64_t* offs, int64_t* mem, int64_t* ri, double* rq, int64_t* ei,
                           double* ed, double* em, int64_t* by) {
  if (!h || !offs || !mem || !ri || !rq || !ei || !ed || !em || !by) return PMMF_INVALID_ARGUMENT;
  auto* r = static_cast<Result*>(h);
  if (s < 0 || s >= static_cast<int64_t>(r->stages.size())) return PMMF_OUT_OF_RANGE;
  const auto& st = r->stages[s];
  std::copy(st.off.begin(), st.off.end(), offs);
  std::copy(st.members.begin(), st.members.end(), mem);
  std::copy(st.rot_idx.begin(), st.rot_idx.end(), ri);
  std::copy(st.rot_q.begin(), st.rot_q.end(), rq);
  std::copy(st.elim_idx.begin(), st.elim_idx.end(), ei);
  std::copy(st.elim_diag.begin(), st.elim_diag.end(), ed);
  std::copy(st.elim_mass.begin(), st.elim_mass.end(), em);
  std::copy(st.bypassed.begin(), st.bypassed.end(), by);
  return PMMF_OK;
}

int pmmf_b200_result_core(void* h, int64_t* ci, double* core, int64_t* di, double* dv) {
  if (!h || !ci || !core || !di || !dv) return PMMF_INVALID_ARGUMENT;
  auto* r = static_cast<Result*>(h);
  std::copy(r->core_idx.begin(), r->core_idx.end(), ci);
  std::copy(r->core.begin(), r->core.end(), core);
  for (size_t i = 0; i < r->diag.size(); ++i) {
    di[i] = r->diag[i].first;
    dv[i] = r->diag[i].second;
  }
  return PMMF_OK;
}

int pmmf_b200_result_stats(void* h, double* phases, int64_t* info) {
  if (!h || !phases || (!info && !static_cast<Result*>(h)->info.empty())) return PMMF_INVALID_ARGUMENT;
  auto* r = static_cast<Result*>(h);
  std::copy(r->phases, r->phases + 6, phases);
  for (size_t s = 0; s < r->info.size(); ++s) std::copy(r->info[s].begin(), r->info[s].end(), info + 7 * s);
  return PMMF_OK;
}

void pmmf_b200_result_free(void* h) { delete static_cast<Result*>(h); }

int pmmf_b200_rotation_from_gram(int32_t k, const double* g, double* q, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (k < 1 || k > kMaxK) fail(PMMF_INVALID_ARGUMENT, "rotation_from_gram: not square");
    double gs[kMaxK][kMaxK], qs[kMaxK][kMaxK];
    for (int a = 0; a < k; ++a)
      for (int b = 0; b < k; ++b) gs[a][b] = g[a * k + b];
    if (k == 1) {
      qs[0][0] = 1.0;
    } else if (!rotation_from_gram(gs, k, qs)) {
      fail(PMMF_INVALID_ARGUMENT, "rotation_from_gram: input not symmetric");
    }
    for (int a = 0; a < k; ++a)
      for (int b = 0; b < k; ++b) q[a * k + b] = qs[a][b];
  });
}

int64_t pmmf_b200_kernel_launches(void) { return launch_counter().load(); }

void pmmf_b200_profile_enable(int32_t on) { prof_set(on != 0); }

int pmmf_b200_profile_read(const char* name, int64_t* launches, double* ms, double* bytes) {
  ProfStat st;
  if (!prof_get(name, &st)) return PMMF_OUT_OF_RANGE;
  *launches = st.launches;
  *ms = st.ms;
  *bytes = st.bytes;
  return PMMF_OK;
}

int64_t pmmf_b200_cached_bytes(int32_t device, int32_t release) {
  int prev = 0;
  if (cudaGetDevice(&prev) != cudaSuccess) return 0;
  if (cudaSetDevice(device) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  if (release) {
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess) {
      BigCache::get().drain(device, s);
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
      try {
        cudaMemPoolTrimTo(lib_pool(device), 0);
      } catch (...) {
      }
    }
    (void)cudaGetLastError();
  }
  int64_t n = 0;
  {
    BigCache& c = BigCache::get();
    std::lock_guard<std::mutex> g(c.mu);
    for (const auto& b : c.blocks)
      if (b.dev == device) n += static_cast<int64_t>(b.bytes);
  }
  cudaSetDevice(prev);
  return n;
}

const char* pmmf_b200_version(void) { return "pmmf_b200 0.1 (sm_100a)"; }

}  // extern "C"
