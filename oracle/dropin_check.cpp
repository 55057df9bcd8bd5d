// oracle/dropin_check.cpp — TEST INFRASTRUCTURE.
// Compiles the C++ drop-in (include/pmmf_b200/dropin.hpp) against the
// reference headers and checks pmmf_b200::factorize == pmmf::factorize and
// GpuOperator::apply == MmfOperator::apply bit-for-bit on a seeded R-MAT
// input (the reference's own operator== on Rotation / Elimination /
// Partition).  Built by oracle/Makefile into oracle/_ref/dropin_check; run
// on the GPU box by tests/test_dropin.py.
#include <pmmf/factorizer.hpp>
#include <pmmf/transform_ops.hpp>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../include/pmmf_b200/dropin.hpp"
#include "../include/pmmf_b200_workloads.h"

int main(int argc, char** argv) {
  const int scale = argc > 1 ? std::atoi(argv[1]) : 11;
  pmmf_b200_workload w{};
  if (pmmf_b200_workload_rmat(scale, 16, 42, 1e-2, &w)) return 2;
  std::vector<pmmf::Triplet> t(static_cast<size_t>(w.nnz));
  for (int64_t i = 0; i < w.nnz; ++i) t[i] = {w.rows[i], w.cols[i], w.vals[i]};
  auto a = pmmf::BlockedSparseMatrix::from_triplets(w.n, t, pmmf::Partition::trivial(w.n));
  pmmf_b200_workload_free(&w);
  pmmf::FactorizeParams p;
  p.cluster.m_target = 16;
  p.seed = 42;
  pmmf::FactorizeStats s_ref, s_gpu;
  const pmmf::MmfFactorization ref = pmmf::factorize(a, p, &s_ref);
  const pmmf::MmfFactorization gpu = pmmf_b200::factorize(a, p, &s_gpu);
  int bad = 0;
  auto check = [&](bool ok, const char* what) {
    if (!ok) {
      std::printf("MISMATCH %s\n", what);
      ++bad;
    }
  };
  check(ref.n == gpu.n, "n");
  check(ref.stages.size() == gpu.stages.size(), "stage count");
  for (size_t s = 0; s < std::min(ref.stages.size(), gpu.stages.size()); ++s) {
    check(*ref.stages[s].partition == *gpu.stages[s].partition, "partition");
    check(ref.stages[s].rotations == gpu.stages[s].rotations, "rotations");
    check(ref.stages[s].eliminated == gpu.stages[s].eliminated, "eliminated");
    check(ref.stages[s].bypassed == gpu.stages[s].bypassed, "bypassed");
  }
  check(ref.h.core_indices == gpu.h.core_indices, "core indices");
  check(ref.h.core == gpu.h.core, "core");
  check(ref.h.diagonal == gpu.h.diagonal, "diagonal");
  check(ref.residual_sq == gpu.residual_sq, "residual_sq");
  check(ref.active_history == gpu.active_history, "active_history");
  check(s_ref.stages.size() == s_gpu.stages.size(), "stats stages");
  // operator
  auto ref_ptr = std::make_shared<const pmmf::MmfFactorization>(ref);
  pmmf::MmfOperator op_ref(ref_ptr);
  pmmf_b200::GpuOperator op_gpu(a, p);
  // the reference's own factorization wrapped on the GPU (no refactorization)
  pmmf_b200::GpuOperator op_wrap(ref_ptr);
  check(&op_wrap.factorization() == ref_ptr.get(), "factorization() identity");
  check(op_gpu.factorization().residual_sq == ref.residual_sq, "factorization() of the GPU operator");
  check(op_wrap.inv_sqrt_zeroed_negatives() == op_ref.inv_sqrt_zeroed_negatives(), "zeroed negatives");
  std::vector<double> v(static_cast<size_t>(a.dim())), o1(v.size()), o2(v.size()), o3(v.size());
  for (size_t i = 0; i < v.size(); ++i) v[i] = std::sin(0.37 * static_cast<double>(i) + 1.0);
  for (auto mode : {pmmf::MmfOperator::Mode::forward, pmmf::MmfOperator::Mode::inverse,
                    pmmf::MmfOperator::Mode::inv_sqrt}) {
    op_ref.apply(mode, v, o1);
    op_gpu.apply(mode, v, o2);
    op_wrap.apply(mode, v, o3);
    check(o1 == o2, "operator apply");
    check(o1 == o3, "wrapped operator apply");
  }
  // a corrupt factorization is rejected as DataError, not a device fault
  {
    pmmf::MmfFactorization corrupt = ref;
    if (!corrupt.stages.empty() && !corrupt.stages[0].rotations.empty()) {
      corrupt.stages[0].rotations[0].indices[0] = corrupt.n + 5;
      bool threw = false;
      try {
        pmmf_b200::GpuOperator op_bad(std::make_shared<const pmmf::MmfFactorization>(corrupt));
      } catch (const pmmf::DataError&) {
        threw = true;
      }
      check(threw, "out-of-range rotation index rejected");
    }
  }
  // solver study: the GPU preconditioners equal the reference's, side by side
  {
    std::vector<double> x(v.size()), r1(v.size()), r2(v.size());
    for (size_t i = 0; i < x.size(); ++i) x[i] = std::cos(0.11 * static_cast<double>(i));
    const pmmf::SplitPreconditioner jr = pmmf::jacobi_preconditioner(a), sr = pmmf::ssor_preconditioner(a, 1.2);
    const pmmf::IncompleteCholesky icr = pmmf::ic_preconditioner(a);
    const pmmf_b200::GpuPreconditioner jg = pmmf_b200::jacobi_preconditioner(a), sg = pmmf_b200::ssor_preconditioner(a, 1.2),
                                       ig = pmmf_b200::ic_preconditioner(a);
    check(ig.compensated() == icr.compensated && ig.alpha() == icr.alpha, "ic compensation");
    const std::pair<const pmmf::SplitPreconditioner*, const pmmf_b200::GpuPreconditioner*> pairs[] = {
        {&jr, &jg}, {&sr, &sg}, {&icr.precond, &ig}};
    for (const auto& [pr, pg] : pairs) {
      const pmmf::SplitPreconditioner k = pg->split();
      pr->left.apply(x, r1);
      k.left.apply(x, r2);
      check(r1 == r2, "preconditioner K^-1");
      pr->right.apply(x, r1);
      pg->apply(1, x, r2);
      check(r1 == r2, "preconditioner K^-T");
    }
    pmmf::SolveConfig sc;
    sc.tol = 1e-8;
    sc.max_iter = 500;
    sc.rhs_count = 2;
    const pmmf::LinearOperator lin = pmmf::make_operator(a);
    const pmmf::SolveReport rr = pmmf::run_solve_experiment(lin, &icr.precond, sc, "ic");
    const pmmf::SolveReport rg = pmmf_b200::run_solve_experiment(a, &ig, sc, "ic");
    check(rr.all_converged == rg.all_converged && std::abs(rr.mean_iterations - rg.mean_iterations) <= 2.0,
          "run_solve_experiment (ic)");
    const pmmf::NystromResult nr = pmmf::nystrom_uniform(a, 64, 9), ng = pmmf_b200::nystrom_uniform(a, 64, 9);
    check(nr.columns == ng.columns && nr.frobenius_error == ng.frobenius_error, "nystrom_uniform");
  }
  std::printf("%s: %zu stages, %zu rotations in stage 1\n", bad ? "FAIL" : "PASS", gpu.stages.size(),
              gpu.stages.empty() ? size_t{0} : gpu.stages[0].rotations.size());
  return bad ? 1 : 0;
}
