// pmmf_b200/dropin.hpp — C++20 drop-in for pmmf::factorize and
// pmmf::MmfOperator on the GPU.
//
// Include AFTER the reference headers (pmmf/factorizer.hpp,
// pmmf/transform_ops.hpp) and link libpmmf_b200.so.  The functions take and
// return the reference's own types, so existing callers only swap the
// namespace:
//
//   pmmf::MmfFactorization f = pmmf_b200::factorize(a, params, &stats);
//       // replaces pmmf::factorize (factorizer.hpp:397-398)
//   auto fp = std::make_shared<const pmmf::MmfFactorization>(std::move(f));
//   pmmf_b200::GpuOperator op(fp);     // replaces pmmf::MmfOperator (transform_ops.hpp:30-41)
//   op.apply(pmmf::MmfOperator::Mode::inv_sqrt, in, out);
//
// GpuOperator wraps any MmfFactorization (from pmmf_b200::factorize, the
// reference's pmmf::factorize or pmmf::load_factorization) without
// refactorizing, exactly as MmfOperator(shared_ptr<const MmfFactorization>,
// zero_threshold) does.
//
// The solver study (solver.hpp:222-416) swaps the same way:
//
//   pmmf_b200::GpuPreconditioner ic = pmmf_b200::ic_preconditioner(a);
//       // replaces pmmf::ic_preconditioner (solver.hpp:278); also jacobi_ /
//       // ssor_ / pmmf_preconditioner
//   pmmf::SolveReport rep = pmmf_b200::run_solve_experiment(a, &ic, cfg, "ic");
//       // replaces pmmf::run_solve_experiment (solver.hpp:368) with CG on the GPU
//   pmmf::SplitPreconditioner k = ic.split();   // or feed the reference's own pcg
//   pmmf::NystromResult ny = pmmf_b200::nystrom_uniform(a, m, seed);
//
// Errors are rethrown as the reference's exception types.
#pragma once

#include <pmmf/factorizer.hpp>
#include <pmmf/solver.hpp>
#include <pmmf/transform_ops.hpp>

#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../pmmf_b200.h"

namespace pmmf_b200 {

inline void rethrow(int status, const char* err) {
  const std::string msg(err);
  switch (status) {
    case PMMF_OK: return;
    case PMMF_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case PMMF_OUT_OF_RANGE: throw std::out_of_range(msg);
    case PMMF_NUMERIC: throw pmmf::NumericError(msg);
    case PMMF_DATA: throw pmmf::DataError(msg);
    default: throw std::runtime_error(msg);
  }
}

struct ResultHandle {
  void* h = nullptr;
  ~ResultHandle() {
    if (h) pmmf_b200_result_free(h);
  }
};

// BlockedSparseMatrix -> triplets + partition (blocked_matrix.hpp:421-436).
inline void to_coo(const pmmf::BlockedSparseMatrix& a, std::vector<int64_t>& r, std::vector<int64_t>& c,
                   std::vector<double>& v, std::vector<int64_t>& off, std::vector<int64_t>& mem) {
  for (const pmmf::Triplet& t : a.to_triplets()) {
    r.push_back(t.row);
    c.push_back(t.col);
    v.push_back(t.value);
  }
  const pmmf::Partition& p = a.partition();
  off.assign(1, 0);
  for (pmmf::index_t u = 0; u < p.num_clusters(); ++u) {
    auto cl = p.cluster(u);
    mem.insert(mem.end(), cl.begin(), cl.end());
    off.push_back(static_cast<int64_t>(mem.size()));
  }
}

inline pmmf_b200_params to_params(const pmmf::FactorizeParams& p) {
  pmmf_b200_params q{};
  q.k = p.k;
  q.n_stages = p.n_stages;
  q.eta = p.eta;
  q.m_target = p.cluster.m_target;
  q.c_min = p.cluster.c_min;
  q.c_max = p.cluster.c_max;
  q.d_max = p.cluster.d_max;
  q.bypass_enabled = p.cluster.bypass_enabled ? 1 : 0;
  q.cluster_seed = p.cluster.seed;
  q.core_min = p.core_min;
  q.core_cap = p.core_cap;
  q.seed = p.seed;
  return q;
}

// Runs the GPU stage loop; returns the raw handle (owned by the caller).
inline void* factorize_handle(const pmmf::BlockedSparseMatrix& input, const pmmf::FactorizeParams& params,
                              int device = 0) {
  std::vector<int64_t> r, c, off, mem;
  std::vector<double> v;
  to_coo(input, r, c, v, off, mem);
  pmmf_b200_coo coo{};
  coo.n = input.dim();
  coo.nnz = static_cast<int64_t>(v.size());
  coo.rows = r.data();
  coo.cols = c.data();
  coo.vals = v.data();
  coo.n_clusters = static_cast<int64_t>(off.size()) - 1;
  coo.cluster_offsets = off.data();
  coo.cluster_members = mem.data();
  coo.on_device = 0;
  coo.device = device;
  const pmmf_b200_params p = to_params(params);
  char err[4096] = {0};
  void* h = nullptr;
  rethrow(pmmf_b200_factorize(&coo, &p, &h, err, sizeof(err)), err);
  return h;
}

// Materialises the reference's MmfFactorization / FactorizeStats
// (factorizer.hpp:56-118) from a result handle.
inline pmmf::MmfFactorization materialize(void* h, const pmmf::FactorizeParams& params,
                                          pmmf::FactorizeStats* stats_out) {
  pmmf_b200_summary s{};
  pmmf_b200_result_summary(h, &s);
  pmmf::MmfFactorization f;
  f.n = s.n;
  f.params = params;
  f.residual_sq = s.residual_sq;
  f.active_history.resize(static_cast<size_t>(s.n_stages + 1));
  pmmf_b200_result_active_history(h, f.active_history.data());
  const int64_t k = s.k;
  for (int64_t st = 0; st < s.n_stages; ++st) {
    pmmf_b200_stage_sizes z{};
    pmmf_b200_result_stage_sizes(h, st, &z);
    std::vector<int64_t> off(z.n_clusters + 1), mem(std::max<int64_t>(z.partition_size, 1)),
        ri(std::max<int64_t>(z.n_rotations * k, 1)), ei(std::max<int64_t>(z.n_eliminated, 1)),
        by(std::max<int64_t>(z.n_bypassed, 1));
    std::vector<double> rq(std::max<int64_t>(z.n_rotations * k * k, 1)), ed(ei.size()), em(ei.size());
    pmmf_b200_result_stage(h, st, off.data(), mem.data(), ri.data(), rq.data(), ei.data(), ed.data(), em.data(),
                           by.data());
    pmmf::Stage stage;
    std::vector<std::vector<pmmf::index_t>> cl;
    for (int64_t u = 0; u < z.n_clusters; ++u) cl.emplace_back(mem.begin() + off[u], mem.begin() + off[u + 1]);
    stage.partition = std::make_shared<const pmmf::Partition>(std::move(cl));
    for (int64_t t = 0; t < z.n_rotations; ++t) {
      pmmf::Rotation rot;
      rot.stage = static_cast<int>(st + 1);
      rot.matrix = pmmf::DenseMatrix(k, k);
      for (int64_t a = 0; a < k; ++a) {
        rot.indices.push_back(ri[t * k + a]);
        for (int64_t b = 0; b < k; ++b) rot.matrix(a, b) = rq[(t * k + a) * k + b];
      }
      stage.rotations.push_back(std::move(rot));
    }
    for (int64_t e = 0; e < z.n_eliminated; ++e) stage.eliminated.push_back({ei[e], ed[e], em[e]});
    stage.bypassed.assign(by.begin(), by.begin() + z.n_bypassed);
    f.stages.push_back(std::move(stage));
  }
  const int64_t g = s.core_size;
  std::vector<int64_t> ci(std::max<int64_t>(g, 1)), di(std::max<int64_t>(s.n_diagonal, 1));
  std::vector<double> core(std::max<int64_t>(g * g, 1)), dv(di.size());
  pmmf_b200_result_core(h, ci.data(), core.data(), di.data(), dv.data());
  f.h.core_indices.assign(ci.begin(), ci.begin() + g);
  f.h.core = pmmf::DenseMatrix(g, g);
  for (int64_t a = 0; a < g; ++a)
    for (int64_t b = 0; b < g; ++b) f.h.core(a, b) = core[a * g + b];
  for (int64_t i = 0; i < s.n_diagonal; ++i) f.h.diagonal.emplace_back(di[i], dv[i]);
  if (stats_out) {
    double ph[6];
    std::vector<int64_t> info(std::max<int64_t>(7 * s.n_stages, 1));
    pmmf_b200_result_stats(h, ph, info.data());
    stats_out->phases = {ph[0], ph[1], ph[2], ph[3], ph[4], ph[5]};
    stats_out->stages.clear();
    for (int64_t st = 0; st < s.n_stages; ++st) {
      const int64_t* o = info.data() + 7 * st;
      stats_out->stages.push_back({static_cast<int>(o[0]), o[1], o[2], o[3], o[4], o[5], static_cast<int>(o[6])});
    }
    stats_out->trivial = s.trivial != 0;
  }
  return f;
}

// Drop-in for pmmf::factorize (factorizer.hpp:397-595).
inline pmmf::MmfFactorization factorize(const pmmf::BlockedSparseMatrix& input, const pmmf::FactorizeParams& params,
                                        pmmf::FactorizeStats* stats_out = nullptr, int device = 0) {
  ResultHandle r;
  r.h = factorize_handle(input, params, device);
  return materialize(r.h, params, stats_out);
}

// The reverse of materialize: a result handle holding an existing
// MmfFactorization (pmmf_b200_result_create / _add_stage / _set_core).
// Throws DataError when the factorization mixes rotation orders (the device
// operator keeps one k per factorization) or holds out-of-range indices.
inline void* result_from(const pmmf::MmfFactorization& f) {
  char err[4096] = {0};
  const int64_t k = f.params.k;
  for (const pmmf::Stage& st : f.stages)
    for (const pmmf::Rotation& rot : st.rotations)
      if (static_cast<int64_t>(rot.indices.size()) != k)
        throw pmmf::DataError("GpuOperator: rotation order differs from params.k");
  const pmmf_b200_params p = to_params(f.params);
  ResultHandle r;
  rethrow(pmmf_b200_result_create(f.n, &p, f.residual_sq, &r.h, err, sizeof(err)), err);
  for (const pmmf::Stage& st : f.stages) {
    std::vector<int64_t> off(1, 0), mem, ri, ei, by(st.bypassed.begin(), st.bypassed.end());
    std::vector<double> rq, ed, em;
    const pmmf::Partition& part = *st.partition;
    for (pmmf::index_t u = 0; u < part.num_clusters(); ++u) {
      auto cl = part.cluster(u);
      mem.insert(mem.end(), cl.begin(), cl.end());
      off.push_back(static_cast<int64_t>(mem.size()));
    }
    for (const pmmf::Rotation& rot : st.rotations) {
      ri.insert(ri.end(), rot.indices.begin(), rot.indices.end());
      for (int64_t a = 0; a < k; ++a)
        for (int64_t b = 0; b < k; ++b) rq.push_back(rot.matrix(a, b));
    }
    for (const pmmf::Elimination& e : st.eliminated) {
      ei.push_back(e.index);
      ed.push_back(e.diagonal);
      em.push_back(e.off_mass_sq);
    }
    rethrow(pmmf_b200_result_add_stage(r.h, static_cast<int64_t>(off.size()) - 1, off.data(), mem.data(),
                                       static_cast<int64_t>(st.rotations.size()), ri.data(), rq.data(),
                                       static_cast<int64_t>(ei.size()), ei.data(), ed.data(), em.data(),
                                       static_cast<int64_t>(by.size()), by.data(), err, sizeof(err)),
            err);
  }
  const int64_t g = static_cast<int64_t>(f.h.core_indices.size());
  std::vector<int64_t> ci(f.h.core_indices.begin(), f.h.core_indices.end()), di;
  std::vector<double> core, dv;
  for (int64_t a = 0; a < g; ++a)
    for (int64_t b = 0; b < g; ++b) core.push_back(f.h.core(a, b));
  for (const auto& [i, d] : f.h.diagonal) {
    di.push_back(i);
    dv.push_back(d);
  }
  std::vector<int64_t> hist(f.active_history.begin(), f.active_history.end());
  rethrow(pmmf_b200_result_set_core(r.h, g, ci.data(), core.data(), static_cast<int64_t>(di.size()), di.data(),
                                    dv.data(), hist.data(), static_cast<int64_t>(hist.size()), err, sizeof(err)),
          err);
  void* h = r.h;
  r.h = nullptr;
  return h;
}

// Drop-in for pmmf::MmfOperator (transform_ops.hpp:30-137) on the GPU.
class GpuOperator {
 public:
  // MmfOperator(shared_ptr<const MmfFactorization>, zero_threshold)
  // (transform_ops.hpp:34-41): the core eigensystem and the rotation stream
  // go to the calling thread's current CUDA device; the factorization is
  // kept for factorization().
  explicit GpuOperator(std::shared_ptr<const pmmf::MmfFactorization> f, double zero_threshold = 1e-12)
      : f_(std::move(f)) {
    if (!f_) throw std::invalid_argument("GpuOperator: null factorization");
    ResultHandle r;
    r.h = result_from(*f_);
    n_ = f_->n;
    char err[4096] = {0};
    rethrow(pmmf_b200_operator_create(r.h, zero_threshold, &op_, err, sizeof(err)), err);
  }
  // Convenience: factorize on the GPU, then wrap (one factorization).
  explicit GpuOperator(const pmmf::BlockedSparseMatrix& input, const pmmf::FactorizeParams& params,
                       double zero_threshold = 1e-12, int device = 0) {
    ResultHandle r;
    r.h = factorize_handle(input, params, device);
    f_ = std::make_shared<const pmmf::MmfFactorization>(materialize(r.h, params, nullptr));
    n_ = input.dim();
    char err[4096] = {0};
    rethrow(pmmf_b200_operator_create(r.h, zero_threshold, &op_, err, sizeof(err)), err);
  }
  const pmmf::MmfFactorization& factorization() const { return *f_; }
  GpuOperator(const GpuOperator&) = delete;
  GpuOperator& operator=(const GpuOperator&) = delete;
  ~GpuOperator() {
    if (op_) pmmf_b200_operator_free(op_);
  }
  pmmf::index_t dim() const { return n_; }
  void* handle() const { return op_; }
  void apply(pmmf::MmfOperator::Mode mode, std::span<const double> in, std::span<double> out) const {
    if (static_cast<pmmf::index_t>(in.size()) != n_ || static_cast<pmmf::index_t>(out.size()) != n_)
      throw std::invalid_argument("MmfOperator::apply: dimension mismatch");
    char err[4096] = {0};
    rethrow(pmmf_b200_operator_apply(op_, static_cast<int32_t>(mode), 1, in.data(), out.data(), 0, err, sizeof(err)),
            err);
  }
  int inv_sqrt_zeroed_negatives() const {
    int64_t v = 0;
    pmmf_b200_operator_zeroed_negatives(op_, &v);
    return static_cast<int>(v);
  }

 private:
  std::shared_ptr<const pmmf::MmfFactorization> f_;
  void* op_ = nullptr;
  pmmf::index_t n_ = 0;
};

// ---- solver study (solver.hpp:222-416) --------------------------------

// A split preconditioner on the GPU (K^-1 = left, K^-T = right).
class GpuPreconditioner {
 public:
  GpuPreconditioner(void* h, pmmf::index_t n) : h_(h, [](void* p) { pmmf_b200_precond_free(p); }), n_(n) {}
  void* handle() const { return h_.get(); }
  pmmf::index_t dim() const { return n_; }
  bool compensated() const {
    int32_t k = 0, c = 0;
    double a = 0.0;
    pmmf_b200_precond_info(h_.get(), &k, &c, &a);
    return c != 0;
  }
  double alpha() const {
    int32_t k = 0, c = 0;
    double a = 0.0;
    pmmf_b200_precond_info(h_.get(), &k, &c, &a);
    return a;
  }
  void apply(int side, std::span<const double> in, std::span<double> out) const {
    if (static_cast<pmmf::index_t>(in.size()) != n_ || static_cast<pmmf::index_t>(out.size()) != n_)
      throw std::invalid_argument("SplitPreconditioner: length mismatch");
    char err[4096] = {0};
    rethrow(pmmf_b200_precond_apply(h_.get(), side, 1, in.data(), out.data(), 0, err, sizeof(err)), err);
  }
  // The reference's own SplitPreconditioner (solver.hpp:49-52) over this handle.
  pmmf::SplitPreconditioner split() const {
    auto h = h_;
    const pmmf::index_t n = n_;
    auto side = [h, n](int s) {
      return [h, n, s](std::span<const double> in, std::span<double> out) {
        char err[4096] = {0};
        rethrow(pmmf_b200_precond_apply(h.get(), s, 1, in.data(), out.data(), 0, err, sizeof(err)), err);
      };
    };
    return {{n, side(0)}, {n, side(1)}};
  }

 private:
  std::shared_ptr<void> h_;
  pmmf::index_t n_;
};

struct CooView {  // owns the triplet arrays behind a pmmf_b200_coo
  std::vector<int64_t> r, c, off, mem;
  std::vector<double> v;
  pmmf_b200_coo coo{};
  CooView(const pmmf::BlockedSparseMatrix& a, int device) {
    to_coo(a, r, c, v, off, mem);
    coo.n = a.dim();
    coo.nnz = static_cast<int64_t>(v.size());
    coo.rows = r.data();
    coo.cols = c.data();
    coo.vals = v.data();
    coo.n_clusters = static_cast<int64_t>(off.size()) - 1;
    coo.cluster_offsets = off.data();
    coo.cluster_members = mem.data();
    coo.device = device;
  }
};

inline GpuPreconditioner make_preconditioner(const pmmf::BlockedSparseMatrix& a, int kind, double omega, int device) {
  CooView cv(a, device);
  char err[4096] = {0};
  void* h = nullptr;
  rethrow(pmmf_b200_precond_create(&cv.coo, kind, omega, &h, err, sizeof(err)), err);
  return GpuPreconditioner(h, a.dim());
}
// jacobi_preconditioner (solver.hpp:222-233)
inline GpuPreconditioner jacobi_preconditioner(const pmmf::BlockedSparseMatrix& a, int device = 0) {
  return make_preconditioner(a, PMMF_PRECOND_JACOBI, 1.0, device);
}
// ssor_preconditioner (solver.hpp:237-267)
inline GpuPreconditioner ssor_preconditioner(const pmmf::BlockedSparseMatrix& a, double omega = 1.0, int device = 0) {
  return make_preconditioner(a, PMMF_PRECOND_SSOR, omega, device);
}
// ic_preconditioner (solver.hpp:278-340); compensated() / alpha() as
// IncompleteCholesky's fields.
inline GpuPreconditioner ic_preconditioner(const pmmf::BlockedSparseMatrix& a, int device = 0) {
  return make_preconditioner(a, PMMF_PRECOND_IC, 1.0, device);
}
// pmmf_preconditioner (solver.hpp:343-349); `op` must outlive the result.
inline GpuPreconditioner pmmf_preconditioner(const GpuOperator& op) {
  char err[4096] = {0};
  void* h = nullptr;
  rethrow(pmmf_b200_precond_from_operator(op.handle(), &h, err, sizeof(err)), err);
  return GpuPreconditioner(h, op.dim());
}

// run_solve_experiment (solver.hpp:368-416) with the CG on the GPU; the
// report is aggregated exactly as the reference aggregates its runs.
inline pmmf::SolveReport run_solve_experiment(const pmmf::BlockedSparseMatrix& a, const GpuPreconditioner* m,
                                              const pmmf::SolveConfig& cfg, const std::string& method_name,
                                              int device = 0) {
  cfg.validate();
  CooView cv(a, device);
  const pmmf_b200_solve_config c{cfg.tol, cfg.max_iter, cfg.rhs_count, cfg.seed};
  const size_t nr = static_cast<size_t>(cfg.rhs_count), stride = static_cast<size_t>(cfg.max_iter) + 1;
  std::vector<int32_t> it(nr), conv(nr), brk(nr);
  std::vector<double> res(nr * stride);
  double wall = 0.0;
  char err[4096] = {0};
  rethrow(pmmf_b200_solve_precond(&cv.coo, m ? m->handle() : nullptr, &c, it.data(), conv.data(), brk.data(),
                                  res.data(), &wall, err, sizeof(err)),
          err);
  pmmf::SolveReport report;
  report.method = method_name;
  report.runs.resize(nr);
  for (size_t r = 0; r < nr; ++r) {
    auto& run = report.runs[r];
    run.iterations = it[r];
    run.converged = conv[r] != 0;
    run.breakdown = brk[r] != 0;
    run.residuals.assign(res.begin() + static_cast<std::ptrdiff_t>(r * stride),
                         res.begin() + static_cast<std::ptrdiff_t>(r * stride + static_cast<size_t>(it[r]) + 1));
  }
  report.wall_ms_total = wall;
  size_t longest = 0;
  long total = 0;
  for (const auto& run : report.runs) {
    longest = std::max(longest, run.residuals.size());
    total += run.iterations;
    report.max_iterations_used = std::max(report.max_iterations_used, run.iterations);
    report.all_converged = report.all_converged && run.converged;
    report.any_breakdown = report.any_breakdown || run.breakdown;
  }
  report.mean_iterations = static_cast<double>(total) / cfg.rhs_count;
  report.per_iteration_ms = total > 0 ? wall / static_cast<double>(total) : 0.0;
  report.mean_residual.assign(longest, 0.0);
  report.std_residual.assign(longest, 0.0);
  for (size_t k = 0; k < longest; ++k) {
    double mean = 0.0;
    for (const auto& run : report.runs) mean += k < run.residuals.size() ? run.residuals[k] : run.residuals.back();
    mean /= cfg.rhs_count;
    double var = 0.0;
    for (const auto& run : report.runs) {
      const double d = (k < run.residuals.size() ? run.residuals[k] : run.residuals.back()) - mean;
      var += d * d;
    }
    report.mean_residual[k] = mean;
    report.std_residual[k] = std::sqrt(var / cfg.rhs_count);
  }
  return report;
}

// nystrom_uniform (transform_ops.hpp:259-307), evaluated on the GPU.
inline pmmf::NystromResult nystrom_uniform(const pmmf::BlockedSparseMatrix& a, pmmf::index_t m, std::uint64_t seed,
                                           pmmf::index_t cap = 4096, int device = 0) {
  CooView cv(a, device);
  pmmf::NystromResult out;
  out.columns.assign(static_cast<size_t>(std::max<pmmf::index_t>(m, 1)), 0);
  char err[4096] = {0};
  rethrow(pmmf_b200_nystrom_uniform(&cv.coo, m, seed, cap, &out.frobenius_error, out.columns.data(), err, sizeof(err)),
          err);
  out.columns.resize(static_cast<size_t>(m));
  return out;
}

}  // namespace pmmf_b200
