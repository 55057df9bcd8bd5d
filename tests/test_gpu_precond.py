"""GPU comparison preconditioners and Nystrom sketch (precond.cu) against the
reference compiled in place (oracle/_ref) and the restatement:

* K^-1 / K^-T of Jacobi, SSOR and IC(0) (solver.hpp:222-340) bit-for-bit —
  the sync-free triangular solves and the IC(0) factorization keep the
  reference's per-entry operation order — plus the compensation decision and
  alpha, and the reference's error cases;
* nystrom_uniform (transform_ops.hpp:252-307): the same sampled columns and a
  bit-identical Frobenius error;
* CG with each preconditioner: the dot products are tree reductions (not the
  reference's sequential sums), so traces agree to the tolerance stated per
  assertion."""
import numpy as np
import pytest

import oracles
import precond_cases as pcs
from cases import api

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", pcs.NAMES)
@pytest.mark.parametrize("kind", ["jacobi", "ssor", "ic"])
@pytest.mark.parametrize("side", [0, 1])
def test_precond_apply_bitwise(name, kind, side):
    inp, part = pcs.build(name)
    vecs = np.random.default_rng(9).standard_normal((37, inp[0]))  # > 32 rhs: two lane rounds per row
    omega = 1.3 if kind == "ssor" else 1.0
    g, ginfo = oracles.precond_apply("gpu", inp, kind, vecs, side, omega, part)
    r, rinfo = oracles.precond_apply("ref", inp, kind, vecs, side, omega, part)
    assert ginfo == rinfo
    assert np.array_equal(g, r)


@pytest.mark.parametrize("kind", ["ssor", "ic"])
def test_precond_apply_large_grid(kind):
    """65,536 rows, 511 dependency levels: the sync-free path at scale."""
    inp = api.workload_aniso_grid(256)
    vecs = np.random.default_rng(1).standard_normal((2, inp[0]))
    for side in (0, 1):
        g, gi = oracles.precond_apply("gpu", inp, kind, vecs, side)
        o, oi = oracles.precond_apply("oracle", inp, kind, vecs, side)
        assert gi == oi
        assert np.array_equal(g, o)


def test_ic_compensated_on_gpu():
    inp, _ = pcs.build("indefinite60")
    _, info = oracles.precond_apply("gpu", inp, "ic", np.ones((1, 60)), 0)
    assert info[1] == 1 and info[2] > 0.0


@pytest.mark.parametrize("kind,omega,inp_fn,code", [
    ("ssor", 2.0, lambda: pcs.build("grid16")[0], 1),
    ("ssor", 1.0, pcs.missing_diagonal, 3),
    ("ic", 1.0, pcs.missing_diagonal, 3),
])
def test_precond_errors(kind, omega, inp_fn, code):
    inp = inp_fn()
    msgs = []
    for which in ("gpu", "ref"):
        with pytest.raises(Exception) as e:
            oracles.precond_apply(which, inp, kind, np.ones((1, inp[0])), 0, omega)
        assert e.value.status == code
        msgs.append(str(e.value))
    assert msgs[0] == msgs[1]


@pytest.mark.parametrize("name,m", [("grid16", 20), ("dense64", 16), ("rmat9", 48), ("rmat9_part", 30),
                                    ("dups_zeros", 144), ("indefinite60", 1), ("grid24_iso", 100)])
def test_nystrom_bitwise(name, m):
    inp, part = pcs.build(name)
    gf, gc = oracles.nystrom("gpu", inp, m, 99, part=part)
    rf, rc = oracles.nystrom("ref", inp, m, 99, part=part)
    assert np.array_equal(gc, rc)
    assert gf == rf


@pytest.mark.parametrize("m,cap,code", [(0, 4096, 1), (257, 4096, 1), (10, 100, 3)])
def test_nystrom_errors(m, cap, code):
    inp, _ = pcs.build("grid16")
    with pytest.raises(Exception) as e:
        oracles.nystrom("gpu", inp, m, 1, cap=cap)
    assert e.value.status == code


@pytest.mark.parametrize("kind", ["none", "jacobi", "ssor", "ic"])
def test_cg_traces_with_preconditioner(kind):
    inp = api.workload_aniso_grid(48)
    gi, gc, gb, gt, _ = oracles.solve_precond("gpu", inp, kind, 1e-8, 3000, 4, 5)
    ri, rc, rb, rt, _ = oracles.solve_precond("ref", inp, kind, 1e-8, 3000, 4, 5)
    assert np.array_equal(gc, rc) and np.array_equal(gb, rb)
    # iteration counts within 2% (rounding of the dot products differs)
    assert np.all(np.abs(gi - ri) <= np.maximum(2, 0.02 * ri)), (gi, ri)
    # the first 20 residuals agree to 1e-9 relative
    assert np.allclose(gt[:, :20], rt[:, :20], rtol=1e-9, atol=0)


def test_python_solver_study_api():
    """The reference's solver-study surface through api.py: every
    preconditioner kind into run_solve_experiment; the pmmf one wraps an
    MmfOperator (solver.hpp:343-349)."""
    from paper_1507_04396_b200 import api as A

    n, r, c, v = api.workload_aniso_grid(32)
    mat = A.BlockedSparseMatrix.from_triplets(n, r, c, v)
    f = A.factorize(mat, A.FactorizeParams(seed=3, cluster=A.ClusterParams(m_target=8)))
    op = A.MmfOperator(f)
    pres = {"none": None, "jacobi": A.jacobi_preconditioner(mat), "ssor": A.ssor_preconditioner(mat, 1.2),
            "ic": A.ic_preconditioner(mat).precond, "pmmf": A.pmmf_preconditioner(op)}
    cfg = A.SolveConfig(tol=1e-8, max_iter=2000, rhs_count=3, seed=1)
    iters = {}
    for name, m in pres.items():
        rep = A.run_solve_experiment(mat, m, cfg, name)
        assert rep.all_converged and not rep.any_breakdown, name
        assert rep.mean_residual[0] == pytest.approx(1.0)
        iters[name] = rep.mean_iterations
    # the pmmf preconditioner through the generic path equals the operator path
    x = np.random.default_rng(0).standard_normal((2, n))
    assert np.array_equal(pres["pmmf"].left(x), op.apply(A.MmfOperator.Mode.inv_sqrt, x))
    assert iters["ic"] < iters["none"] and iters["ssor"] < iters["none"]
    ny = A.nystrom_uniform(mat, 64, 5)
    assert len(ny.columns) == 64 and ny.frobenius_error > 0.0
