"""CPU: the restated comparison preconditioners and Nystrom sketch
(oracle/liboracle.so) are pinned bit-for-bit to the reference compiled in
place (oracle/_ref: jacobi/ssor/ic_preconditioner, solver.hpp:222-340;
nystrom_uniform, transform_ops.hpp:252-307), including the IC(0)
compensation decision and alpha, and the reference's error cases."""
import numpy as np
import pytest

import oracles
import precond_cases as pcs
from paper_1507_04396_b200 import abi

needs_ref = pytest.mark.skipif(not oracles.available("ref"), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("name", pcs.NAMES)
@pytest.mark.parametrize("kind", ["jacobi", "ssor", "ic"])
@pytest.mark.parametrize("side", [0, 1])
def test_precond_restatement_matches_reference(name, kind, side):
    inp, part = pcs.build(name)
    vecs = np.random.default_rng(5).standard_normal((3, inp[0]))
    omega = 1.3 if kind == "ssor" else 1.0
    r, rinfo = oracles.precond_apply("ref", inp, kind, vecs, side, omega, part)
    o, oinfo = oracles.precond_apply("oracle", inp, kind, vecs, side, omega, part)
    assert rinfo == oinfo
    assert np.array_equal(r, o)


@needs_ref
def test_ic_compensation_is_exercised():
    inp, part = pcs.build("indefinite60")
    _, info = oracles.precond_apply("ref", inp, "ic", np.ones((1, 60)), 0)
    assert info[1] == 1 and info[2] > 0.0


@needs_ref
@pytest.mark.parametrize("kind,omega,inp_fn,code", [
    ("ssor", 2.0, lambda: pcs.build("grid16")[0], 1),
    ("ssor", 0.0, lambda: pcs.build("grid16")[0], 1),
    ("ssor", 1.0, pcs.missing_diagonal, 3),
    ("ic", 1.0, pcs.missing_diagonal, 3),
])
def test_precond_errors_match_reference(kind, omega, inp_fn, code):
    inp = inp_fn()
    msgs = []
    for which in ("ref", "oracle"):
        with pytest.raises(abi.PmmfError) as e:
            oracles.precond_apply(which, inp, kind, np.ones((1, inp[0])), 0, omega)
        assert e.value.status == code
        msgs.append(str(e.value))
    assert msgs[0] == msgs[1]


@needs_ref
@pytest.mark.parametrize("name,m", [("grid16", 20), ("dense64", 16), ("rmat9", 48), ("rmat9_part", 30),
                                    ("dups_zeros", 144), ("indefinite60", 1)])
def test_nystrom_restatement_matches_reference(name, m):
    inp, part = pcs.build(name)
    rf, rc = oracles.nystrom("ref", inp, m, 99, part=part)
    of, oc = oracles.nystrom("oracle", inp, m, 99, part=part)
    assert np.array_equal(rc, oc)
    assert rf == of


@needs_ref
@pytest.mark.parametrize("m,cap,code", [(0, 4096, 1), (257, 4096, 1),
                                        (10, 100, 3)])
def test_nystrom_errors_match_reference(m, cap, code):
    inp, _ = pcs.build("grid16")
    for which in ("ref", "oracle"):
        with pytest.raises(abi.PmmfError) as e:
            oracles.nystrom(which, inp, m, 1, cap=cap)
        assert e.value.status == code


@needs_ref
@pytest.mark.parametrize("kind", ["none", "jacobi", "ssor", "ic"])
def test_solve_restatement_matches_reference(kind):
    inp, _ = pcs.build("grid16")
    ri, rc, rb, rt, _ = oracles.solve_precond("ref", inp, kind, 1e-8, 400, 3, 5)
    oi, oc, ob, ot, _ = oracles.solve_precond("oracle", inp, kind, 1e-8, 400, 3, 5)
    assert np.array_equal(ri, oi) and np.array_equal(rc, oc) and np.array_equal(rb, ob)
    assert np.array_equal(np.nan_to_num(rt, nan=-1.0), np.nan_to_num(ot, nan=-1.0))
