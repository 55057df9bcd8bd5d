"""CPU: libpmmf_b200.so (sm_100a fatbin, C-ABI) loads without a GPU and
exports every entry point declared in include/*.h; the workload generators
reproduce the SURVEY.md §8(d) recipe counts; errors map onto the reference's
exception taxonomy."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1507_04396_b200 import abi, api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = []
    for h in ["pmmf_b200.h", "pmmf_b200_workloads.h"]:
        txt = open(os.path.join(ROOT, "include", h)).read()
        syms += re.findall(r"\b(pmmf_b200_[a-z0-9_]+)\s*\(", txt)
    return sorted(set(syms))


def test_exports_every_declared_symbol():
    lib = api.library().lib
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s


def test_library_is_built_for_sm100a():
    out = os.popen(f"cuobjdump --list-elf {api.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def test_version_and_launch_counter():
    L = api.library().lib
    assert b"sm_100a" in L.pmmf_b200_version()
    assert L.pmmf_b200_kernel_launches() >= 0


@pytest.mark.parametrize("scale,epv,nnz", [(16, 16, 1020912), (18, 32, 7873696)])
def test_rmat_recipe_counts(scale, epv, nnz):
    n, r, c, v = api.workload_rmat(scale, epv, 42)
    assert n == 1 << scale and len(v) == nnz
    assert np.all(np.isfinite(v))


def test_grid_recipe_count():
    n, r, c, v = api.workload_aniso_grid(1024)
    assert n == 1 << 20 and len(v) == 5238784


def test_rhs_generator_matches_reference_solver_rhs():
    # run_solve_experiment (solver.hpp:375-381): unit norm
    out = np.zeros(2 * 100)
    api.library().lib.pmmf_b200_workload_rhs(ctypes.c_int64(100), ctypes.c_int32(2), ctypes.c_uint64(5),
                                             out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    b = out.reshape(2, 100)
    assert np.allclose(np.linalg.norm(b, axis=1), 1.0, atol=1e-15)


def test_error_mapping_types():
    assert issubclass(abi.InvalidArgument, ValueError)
    assert issubclass(abi.OutOfRange, IndexError)
    with pytest.raises(abi.NumericError):
        abi.raise_for(3, ctypes.create_string_buffer(b"x"))


def test_header_is_plain_c(tmp_path):
    """include/pmmf_b200.h is the drop-in boundary for cgo/ctypes/C callers:
    it must compile as strict C99 with no C++ types."""
    import shutil
    import subprocess

    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        import pytest

        pytest.skip("no C compiler")
    src = tmp_path / "h.c"
    src.write_text('#include "pmmf_b200.h"\nint main(void) { return (int)sizeof(pmmf_b200_triplets) == 0; }\n')
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    r = subprocess.run([cc, "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I", inc, "-c", str(src), "-o",
                        str(tmp_path / "h.o")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
