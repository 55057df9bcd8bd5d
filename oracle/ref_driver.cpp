// oracle/ref_driver.cpp — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// Exposes the UNMODIFIED reference implementation (header-only C++20 under
// /root/reference/proj/include/pmmf, compiled in place by oracle/Makefile)
// through the same flat C-ABI shape as include/pmmf_b200.h, with the prefix
// pmmf_ref_ instead of pmmf_b200_.  Built into oracle/_ref/libpmmf_ref.so.
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
// --impl reference) may load it, and only as the checker / CPU baseline.
//
// Nothing here re-implements the algorithm: every call forwards to the
// reference (pmmf::factorize, pmmf::MmfOperator, pmmf::run_solve_experiment,
// pmmf::rotation_from_gram, pmmf::residual_frobenius, and the input path
// pmmf::read_matrix_market / read_edge_list / write_matrix_market /
// laplacian / symmetrize of io.hpp).

#include <pmmf/blocked_matrix.hpp>
#include <pmmf/factorizer.hpp>
#include <pmmf/io.hpp>
#include <pmmf/parallel.hpp>
#include <pmmf/solver.hpp>
#include <pmmf/transform_ops.hpp>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "../include/pmmf_b200.h"
#include "../include/pmmf_b200_workloads.h"
#include "../paper_1507_04396_b200/csrc/recipes.hpp"

namespace {

struct RefResult {
  std::shared_ptr<pmmf::MmfFactorization> f;
  pmmf::FactorizeStats stats;
};

struct RefOperator {
  std::shared_ptr<pmmf::MmfOperator> op;
};

void set_err(char* err, size_t errlen, const std::string& msg) {
  if (!err || errlen == 0) return;
  std::size_t n = std::min(errlen - 1, msg.size());
  std::memcpy(err, msg.data(), n);
  err[n] = '\0';
}

template <typename Fn>
int guarded(char* err, size_t errlen, Fn&& fn) {
  try {
    fn();
    return PMMF_OK;
  } catch (const std::invalid_argument& e) {
    set_err(err, errlen, e.what());
    return PMMF_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    set_err(err, errlen, e.what());
    return PMMF_OUT_OF_RANGE;
  } catch (const pmmf::NumericError& e) {
    set_err(err, errlen, e.what());
    return PMMF_NUMERIC;
  } catch (const pmmf::DataError& e) {
    set_err(err, errlen, e.what());
    return PMMF_DATA;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return PMMF_INTERNAL;
  }
}

pmmf::Partition make_partition(const pmmf_b200_coo* a) {
  if (a->n_clusters == 0) return pmmf::Partition::trivial(a->n);
  std::vector<std::vector<pmmf::index_t>> clusters(static_cast<std::size_t>(a->n_clusters));
  for (int64_t u = 0; u < a->n_clusters; ++u)
    clusters[static_cast<std::size_t>(u)].assign(a->cluster_members + a->cluster_offsets[u],
                                                 a->cluster_members + a->cluster_offsets[u + 1]);
  return pmmf::Partition(std::move(clusters));
}

pmmf::BlockedSparseMatrix make_matrix(const pmmf_b200_coo* a) {
  if (a->on_device) throw std::invalid_argument("reference path takes host buffers only");
  std::vector<pmmf::Triplet> t(static_cast<std::size_t>(a->nnz));
  for (int64_t i = 0; i < a->nnz; ++i) t[static_cast<std::size_t>(i)] = {a->rows[i], a->cols[i], a->vals[i]};
  return pmmf::BlockedSparseMatrix::from_triplets(a->n, t, make_partition(a));
}

pmmf::FactorizeParams make_params(const pmmf_b200_params* p) {
  pmmf::FactorizeParams fp;
  fp.k = p->k;
  fp.n_stages = p->n_stages;
  fp.eta = p->eta;
  fp.cluster.m_target = p->m_target;
  fp.cluster.c_min = p->c_min;
  fp.cluster.c_max = p->c_max;
  fp.cluster.d_max = p->d_max;
  fp.cluster.bypass_enabled = p->bypass_enabled != 0;
  fp.cluster.seed = p->cluster_seed;
  fp.core_min = p->core_min;
  fp.core_cap = p->core_cap;
  fp.seed = p->seed;
  return fp;
}

}  // namespace

extern "C" {

void pmmf_ref_set_threads(int32_t n) { pmmf::parallel::set_max_threads(n); }

int pmmf_ref_factorize(const pmmf_b200_coo* a, const pmmf_b200_params* p, void** out, char* err,
                       size_t errlen) {
  return guarded(err, errlen, [&] {
    auto m = make_matrix(a);
    auto r = std::make_unique<RefResult>();
    r->f = std::make_shared<pmmf::MmfFactorization>(pmmf::factorize(m, make_params(p), &r->stats));
    *out = r.release();
  });
}

int pmmf_ref_result_summary(void* h, pmmf_b200_summary* out) {
  auto* r = static_cast<RefResult*>(h);
  const auto& f = *r->f;
  out->n = f.n;
  out->n_stages = static_cast<int64_t>(f.stages.size());
  out->k = f.params.k;
  out->core_size = static_cast<int64_t>(f.h.core_indices.size());
  out->n_diagonal = static_cast<int64_t>(f.h.diagonal.size());
  out->trivial = r->stats.trivial ? 1 : 0;
  out->residual_sq = f.residual_sq;
  return PMMF_OK;
}

int pmmf_ref_result_active_history(void* h, int64_t* out) {
  const auto& f = *static_cast<RefResult*>(h)->f;
  for (std::size_t i = 0; i < f.active_history.size(); ++i) out[i] = f.active_history[i];
  return PMMF_OK;
}

int pmmf_ref_result_stage_sizes(void* h, int64_t s, pmmf_b200_stage_sizes* out) {
  const auto& f = *static_cast<RefResult*>(h)->f;
  if (s < 0 || s >= static_cast<int64_t>(f.stages.size())) return PMMF_OUT_OF_RANGE;
  const auto& st = f.stages[static_cast<std::size_t>(s)];
  out->n_clusters = st.partition->num_clusters();
  out->partition_size = st.partition->size();
  out->n_rotations = static_cast<int64_t>(st.rotations.size());
  out->n_eliminated = static_cast<int64_t>(st.eliminated.size());
  out->n_bypassed = static_cast<int64_t>(st.bypassed.size());
  return PMMF_OK;
}

int pmmf_ref_result_stage(void* h, int64_t s, int64_t* cluster_offsets, int64_t* members,
                          int64_t* rot_indices, double* rot_matrices, int64_t* elim_index,
                          double* elim_diagonal, double* elim_off_mass_sq, int64_t* bypassed) {
  const auto& f = *static_cast<RefResult*>(h)->f;
  if (s < 0 || s >= static_cast<int64_t>(f.stages.size())) return PMMF_OUT_OF_RANGE;
  const auto& st = f.stages[static_cast<std::size_t>(s)];
  int64_t pos = 0;
  cluster_offsets[0] = 0;
  for (int64_t u = 0; u < st.partition->num_clusters(); ++u) {
    for (auto g : st.partition->cluster(u)) members[pos++] = g;
    cluster_offsets[u + 1] = pos;
  }
  const int64_t k = f.params.k;
  for (std::size_t t = 0; t < st.rotations.size(); ++t) {
    const auto& rot = st.rotations[t];
    for (int64_t a = 0; a < k; ++a) {
      rot_indices[static_cast<int64_t>(t) * k + a] = rot.indices[static_cast<std::size_t>(a)];
      for (int64_t b = 0; b < k; ++b) rot_matrices[(static_cast<int64_t>(t) * k + a) * k + b] = rot.matrix(a, b);
    }
  }
  for (std::size_t e = 0; e < st.eliminated.size(); ++e) {
    elim_index[e] = st.eliminated[e].index;
    elim_diagonal[e] = st.eliminated[e].diagonal;
    elim_off_mass_sq[e] = st.eliminated[e].off_mass_sq;
  }
  for (std::size_t b = 0; b < st.bypassed.size(); ++b) bypassed[b] = st.bypassed[b];
  return PMMF_OK;
}

int pmmf_ref_result_core(void* h, int64_t* core_indices, double* core, int64_t* diag_index,
                         double* diag_value) {
  const auto& f = *static_cast<RefResult*>(h)->f;
  const auto g = static_cast<int64_t>(f.h.core_indices.size());
  for (int64_t a = 0; a < g; ++a) {
    core_indices[a] = f.h.core_indices[static_cast<std::size_t>(a)];
    for (int64_t b = 0; b < g; ++b) core[a * g + b] = f.h.core(a, b);
  }
  for (std::size_t i = 0; i < f.h.diagonal.size(); ++i) {
    diag_index[i] = f.h.diagonal[i].first;
    diag_value[i] = f.h.diagonal[i].second;
  }
  return PMMF_OK;
}

int pmmf_ref_result_stats(void* h, double* phases, int64_t* stage_info) {
  const auto& st = static_cast<RefResult*>(h)->stats;
  phases[0] = st.phases.clustering_ms;
  phases[1] = st.phases.gram_ms;
  phases[2] = st.phases.rotations_ms;
  phases[3] = st.phases.apply_ms;
  phases[4] = st.phases.reblocking_ms;
  phases[5] = st.phases.total_ms;
  for (std::size_t s = 0; s < st.stages.size(); ++s) {
    const auto& i = st.stages[s];
    int64_t* o = stage_info + 7 * s;
    o[0] = i.stage;
    o[1] = i.clusters;
    o[2] = i.bypassed;
    o[3] = i.rotations;
    o[4] = i.eliminated;
    o[5] = i.active_after;
    o[6] = i.cluster_recursion_depth;
  }
  return PMMF_OK;
}

void pmmf_ref_result_free(void* h) { delete static_cast<RefResult*>(h); }

int pmmf_ref_operator_create(void* result, double zero_threshold, void** op, char* err,
                             size_t errlen) {
  return guarded(err, errlen, [&] {
    auto* r = static_cast<RefResult*>(result);
    auto o = std::make_unique<RefOperator>();
    o->op = std::make_shared<pmmf::MmfOperator>(r->f, zero_threshold);
    *op = o.release();
  });
}

int pmmf_ref_operator_apply(void* op, int32_t mode, int64_t nrhs, const double* in, double* out,
                            int32_t on_device, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (on_device) throw std::invalid_argument("reference path takes host buffers only");
    auto* o = static_cast<RefOperator*>(op);
    const auto n = static_cast<std::size_t>(o->op->dim());
    const auto m = static_cast<pmmf::MmfOperator::Mode>(mode);
    pmmf::parallel::for_each_index(static_cast<std::size_t>(nrhs), [&](std::size_t r) {
      o->op->apply(m, std::span<const double>(in + r * n, n), std::span<double>(out + r * n, n));
    });
  });
}

int pmmf_ref_operator_zeroed_negatives(void* op, int64_t* out) {
  *out = static_cast<RefOperator*>(op)->op->inv_sqrt_zeroed_negatives();
  return PMMF_OK;
}

void pmmf_ref_operator_free(void* op) { delete static_cast<RefOperator*>(op); }

int pmmf_ref_solve(const pmmf_b200_coo* a, void* op, const pmmf_b200_solve_config* cfg,
                   int32_t* iterations, int32_t* converged, int32_t* breakdown, double* residuals,
                   double* wall_ms, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    auto m = make_matrix(a);
    pmmf::LinearOperator lin = pmmf::make_operator(m);
    pmmf::SolveConfig sc;
    sc.tol = cfg->tol;
    sc.max_iter = cfg->max_iter;
    sc.rhs_count = cfg->rhs_count;
    sc.seed = cfg->seed;
    pmmf::SolveReport rep;
    if (op) {
      auto* o = static_cast<RefOperator*>(op);
      auto f = std::shared_ptr<const pmmf::MmfFactorization>(&o->op->factorization(),
                                                             [](const pmmf::MmfFactorization*) {});
      pmmf::SplitPreconditioner pre = pmmf::pmmf_preconditioner(f);
      rep = pmmf::run_solve_experiment(lin, &pre, sc, "pmmf");
    } else {
      rep = pmmf::run_solve_experiment(lin, nullptr, sc, "none");
    }
    const int64_t stride = cfg->max_iter + 1;
    for (int r = 0; r < cfg->rhs_count; ++r) {
      const auto& run = rep.runs[static_cast<std::size_t>(r)];
      iterations[r] = run.iterations;
      converged[r] = run.converged ? 1 : 0;
      breakdown[r] = run.breakdown ? 1 : 0;
      for (int64_t i = 0; i < stride; ++i)
        residuals[r * stride + i] =
            i < static_cast<int64_t>(run.residuals.size()) ? run.residuals[static_cast<std::size_t>(i)] : NAN;
    }
    *wall_ms = rep.wall_ms_total;
  });
}

// ---- comparison preconditioners (solver.hpp:222-349), the reference's own
struct RefPrecond {
  pmmf::SplitPreconditioner pre;
  int kind = 0;
  int64_t n = 0;
  int compensated = 0;
  double alpha = 0.0;
};

int pmmf_ref_precond_create(const pmmf_b200_coo* a, int32_t kind, double omega, void** out, char* err,
                            size_t errlen) {
  return guarded(err, errlen, [&] {
    auto m = make_matrix(a);
    auto p = std::make_unique<RefPrecond>();
    p->kind = kind;
    p->n = a->n;
    if (kind == PMMF_PRECOND_JACOBI) {
      p->pre = pmmf::jacobi_preconditioner(m);
    } else if (kind == PMMF_PRECOND_SSOR) {
      p->pre = pmmf::ssor_preconditioner(m, omega);
    } else if (kind == PMMF_PRECOND_IC) {
      pmmf::IncompleteCholesky ic = pmmf::ic_preconditioner(m);
      p->pre = ic.precond;
      p->compensated = ic.compensated ? 1 : 0;
      p->alpha = ic.alpha;
    } else {
      throw std::invalid_argument("preconditioner: unknown kind");
    }
    *out = p.release();
  });
}

int pmmf_ref_precond_from_operator(void* op, void** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    auto* o = static_cast<RefOperator*>(op);
    auto f = std::shared_ptr<const pmmf::MmfFactorization>(&o->op->factorization(),
                                                           [](const pmmf::MmfFactorization*) {});
    auto p = std::make_unique<RefPrecond>();
    p->kind = PMMF_PRECOND_PMMF;
    p->n = o->op->dim();
    p->pre = pmmf::pmmf_preconditioner(f);
    *out = p.release();
  });
}

int pmmf_ref_precond_apply(void* pc, int32_t side, int64_t nrhs, const double* in, double* out, int32_t on_device,
                           char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (on_device) throw std::invalid_argument("reference path takes host buffers only");
    auto* p = static_cast<RefPrecond*>(pc);
    const auto n = static_cast<std::size_t>(p->n);
    const pmmf::LinearOperator& op = side == 0 ? p->pre.left : p->pre.right;
    for (int64_t r = 0; r < nrhs; ++r)
      op.apply(std::span<const double>(in + r * n, n), std::span<double>(out + r * n, n));
  });
}

int pmmf_ref_precond_info(void* pc, int32_t* kind, int32_t* compensated, double* alpha) {
  auto* p = static_cast<RefPrecond*>(pc);
  *kind = p->kind;
  *compensated = p->compensated;
  *alpha = p->alpha;
  return PMMF_OK;
}

void pmmf_ref_precond_free(void* pc) { delete static_cast<RefPrecond*>(pc); }

int pmmf_ref_solve_precond(const pmmf_b200_coo* a, void* pc, const pmmf_b200_solve_config* cfg,
                           int32_t* iterations, int32_t* converged, int32_t* breakdown, double* residuals,
                           double* wall_ms, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    auto m = make_matrix(a);
    pmmf::LinearOperator lin = pmmf::make_operator(m);
    pmmf::SolveConfig sc;
    sc.tol = cfg->tol;
    sc.max_iter = cfg->max_iter;
    sc.rhs_count = cfg->rhs_count;
    sc.seed = cfg->seed;
    auto* p = static_cast<RefPrecond*>(pc);
    pmmf::SolveReport rep = pmmf::run_solve_experiment(lin, p ? &p->pre : nullptr, sc, "precond");
    const int64_t stride = cfg->max_iter + 1;
    for (int r = 0; r < cfg->rhs_count; ++r) {
      const auto& run = rep.runs[static_cast<std::size_t>(r)];
      iterations[r] = run.iterations;
      converged[r] = run.converged ? 1 : 0;
      breakdown[r] = run.breakdown ? 1 : 0;
      for (int64_t i = 0; i < stride; ++i)
        residuals[r * stride + i] =
            i < static_cast<int64_t>(run.residuals.size()) ? run.residuals[static_cast<std::size_t>(i)] : NAN;
    }
    *wall_ms = rep.wall_ms_total;
  });
}

int pmmf_ref_nystrom_uniform(const pmmf_b200_coo* a, int64_t m, uint64_t seed, int64_t cap, double* fro,
                             int64_t* columns, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    auto mat = make_matrix(a);
    pmmf::NystromResult r = pmmf::nystrom_uniform(mat, m, seed, cap);
    *fro = r.frobenius_error;
    std::copy(r.columns.begin(), r.columns.end(), columns);
  });
}

int pmmf_ref_rotation_from_gram(int32_t k, const double* g, double* q, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    pmmf::DenseMatrix gs(k, k);
    for (int a = 0; a < k; ++a)
      for (int b = 0; b < k; ++b) gs(a, b) = g[a * k + b];
    pmmf::DenseMatrix qm = pmmf::rotation_from_gram(gs);
    for (int a = 0; a < k; ++a)
      for (int b = 0; b < k; ++b) q[a * k + b] = qm(a, b);
  });
}

// Dense reconstruction error ||A - Q^T H Q||_F (transform_ops.hpp:225-237),
// both methods; n <= cap only.
int pmmf_ref_residual_frobenius(void* result, const pmmf_b200_coo* a, double* accumulated,
                                double* dense, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    auto m = make_matrix(a);
    const auto& f = *static_cast<RefResult*>(result)->f;
    *accumulated = pmmf::residual_frobenius(f, m, pmmf::ResidualMethod::accumulated);
    *dense = pmmf::residual_frobenius(f, m, pmmf::ResidualMethod::dense);
  });
}

static pmmf_b200_triplets* ref_triplets(pmmf::index_t rows, pmmf::index_t cols, const std::vector<pmmf::Triplet>& t,
                                        const std::vector<pmmf::index_t>* ids) {
  auto* o = static_cast<pmmf_b200_triplets*>(std::calloc(1, sizeof(pmmf_b200_triplets)));
  o->rows = rows;
  o->cols = cols;
  o->nnz = static_cast<int64_t>(t.size());
  const size_t n = std::max<size_t>(t.size(), 1);
  o->row = static_cast<int64_t*>(std::malloc(n * sizeof(int64_t)));
  o->col = static_cast<int64_t*>(std::malloc(n * sizeof(int64_t)));
  o->val = static_cast<double*>(std::malloc(n * sizeof(double)));
  for (size_t i = 0; i < t.size(); ++i) {
    o->row[i] = t[i].row;
    o->col[i] = t[i].col;
    o->val[i] = t[i].value;
  }
  if (ids) {
    o->n_ids = static_cast<int64_t>(ids->size());
    o->original_ids = static_cast<int64_t*>(std::malloc(std::max<size_t>(ids->size(), 1) * sizeof(int64_t)));
    for (size_t i = 0; i < ids->size(); ++i) o->original_ids[i] = (*ids)[i];
  }
  return o;
}

void pmmf_ref_triplets_free(pmmf_b200_triplets* t) {
  if (!t) return;
  std::free(t->row);
  std::free(t->col);
  std::free(t->val);
  std::free(t->original_ids);
  std::free(t);
}

int pmmf_ref_read_matrix_market(const char* path, pmmf_b200_triplets** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    const pmmf::TripletMatrix m = pmmf::read_matrix_market(std::string(path));
    *out = ref_triplets(m.rows, m.cols, m.entries, nullptr);
  });
}

int pmmf_ref_read_edge_list(const char* path, pmmf_b200_triplets** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    const pmmf::EdgeList e = pmmf::read_edge_list(std::string(path));
    *out = ref_triplets(e.n, e.n, e.entries, &e.original_ids);
  });
}

static std::vector<pmmf::Triplet> ref_in(int64_t nnz, const int64_t* r, const int64_t* c, const double* v) {
  std::vector<pmmf::Triplet> t(static_cast<size_t>(nnz));
  for (int64_t i = 0; i < nnz; ++i) t[i] = {r[i], c[i], v[i]};
  return t;
}

int pmmf_ref_write_matrix_market(const char* path, int64_t rows, int64_t cols, int64_t nnz, const int64_t* r,
                                 const int64_t* c, const double* v, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    const auto t = ref_in(nnz, r, c, v);
    pmmf::write_matrix_market(std::string(path), rows, cols, t);
  });
}

int pmmf_ref_laplacian(int64_t n, int64_t nnz, const int64_t* r, const int64_t* c, const double* v, double shift,
                       int64_t* out_r, int64_t* out_c, double* out_v, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    const auto t = ref_in(nnz, r, c, v);
    const auto o = pmmf::laplacian(t, n, shift);
    for (size_t i = 0; i < o.size(); ++i) {
      out_r[i] = o[i].row;
      out_c[i] = o[i].col;
      out_v[i] = o[i].value;
    }
  });
}

int pmmf_ref_symmetrize(int64_t nnz, const int64_t* r, const int64_t* c, const double* v, int64_t* out_nnz,
                        int64_t* out_r, int64_t* out_c, double* out_v, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    const auto t = ref_in(nnz, r, c, v);
    const auto o = pmmf::symmetrize(t);
    *out_nnz = static_cast<int64_t>(o.size());
    for (size_t i = 0; i < o.size(); ++i) {
      out_r[i] = o[i].row;
      out_c[i] = o[i].col;
      out_v[i] = o[i].value;
    }
  });
}

// ---- seeded inputs on the reference's own generator (pmmf::Rng, rng.hpp) ----
// The recipes of SURVEY.md §8(d) (paper_1507_04396_b200/csrc/recipes.hpp,
// templates over the draw interface) instantiated on pmmf::Rng, so the
// --impl reference arm of bench.py never loads libpmmf_b200.so.

static int ref_emit(const pmmf_recipes::Coo& coo, pmmf_b200_workload* out) {
  const size_t m = coo.v.size();
  out->n = coo.n;
  out->nnz = static_cast<int64_t>(m);
  out->rows = static_cast<int64_t*>(std::malloc(std::max<size_t>(1, m) * sizeof(int64_t)));
  out->cols = static_cast<int64_t*>(std::malloc(std::max<size_t>(1, m) * sizeof(int64_t)));
  out->vals = static_cast<double*>(std::malloc(std::max<size_t>(1, m) * sizeof(double)));
  if (!out->rows || !out->cols || !out->vals) return 1;
  if (m) {
    std::memcpy(out->rows, coo.r.data(), m * sizeof(int64_t));
    std::memcpy(out->cols, coo.c.data(), m * sizeof(int64_t));
    std::memcpy(out->vals, coo.v.data(), m * sizeof(double));
  }
  return 0;
}

int pmmf_ref_workload_rmat(int32_t scale, int32_t epv, uint64_t seed, double shift, pmmf_b200_workload* out) {
  pmmf::Rng rng(seed);
  pmmf_recipes::Coo coo;
  return pmmf_recipes::rmat(scale, epv, rng, shift, coo) ? ref_emit(coo, out) : 1;
}

int pmmf_ref_workload_dense_spd(int64_t n, int64_t d, uint64_t seed, double shift, pmmf_b200_workload* out) {
  pmmf::Rng rng(seed);
  pmmf_recipes::Coo coo;
  return pmmf_recipes::dense_spd(n, d, rng, shift, coo) ? ref_emit(coo, out) : 1;
}

int pmmf_ref_workload_rbf(int64_t n, int32_t dim, double bw, uint64_t seed, double shift, pmmf_b200_workload* out) {
  pmmf::Rng rng(seed);
  pmmf_recipes::Coo coo;
  return pmmf_recipes::rbf(n, dim, bw, rng, shift, coo) ? ref_emit(coo, out) : 1;
}

int pmmf_ref_workload_aniso_grid(int64_t side, double ax, double ay, pmmf_b200_workload* out) {
  pmmf_recipes::Coo coo;
  return pmmf_recipes::aniso_grid(side, ax, ay, coo) ? ref_emit(coo, out) : 1;
}

void pmmf_ref_workload_free(pmmf_b200_workload* w) {
  if (!w) return;
  std::free(w->rows);
  std::free(w->cols);
  std::free(w->vals);
  w->rows = w->cols = nullptr;
  w->vals = nullptr;
}

}  // extern "C"
