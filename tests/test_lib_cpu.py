"""CPU: the C-ABI library loads, exports exactly what include/ibmgpu.h declares, and the Python
mirror keeps the reference's names and argument validation. No compute calls (no GPU here)."""
import ctypes as C
import os
import subprocess

import pytest

from paper_1109_3524_b200 import _lib, ibm


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    declared = _lib.header_symbols()
    assert len(declared) >= 50
    for name in declared:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T ibmgpu_" in ln}
    assert set(declared) == exported


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_string():
    assert b"sm_100a" in _lib.load().ibmgpu_version()


def test_python_mirror_names():
    for name in ("SparseMatrix", "spmm", "sliced_triple_product", "add_sparse", "symmetrized", "pin_row_col",
                 "is_symmetric", "pcg", "cg", "IdentityPreconditioner", "DiagonalPreconditioner", "SaPreconditioner",
                 "SaOptions", "build_sa_hierarchy", "sa_apply", "amg_solve", "assemble_coupled_system",
                 "assemble_interpolation_regularization", "delta_roma", "Stepper", "SolverParams"):
        assert hasattr(ibm, name), name


def test_solver_params_validation():
    # krylov.hpp:21-24
    p = ibm.SolverParams(rel_tol=2.0)
    with pytest.raises(ValueError):
        p.validate()
    p = ibm.SolverParams(max_iters=0)
    with pytest.raises(ValueError):
        p.validate()
    ibm.SolverParams().validate()


def test_no_cpu_fallback_without_device():
    """Without a CUDA device the product must fail loudly, not compute on the CPU."""
    if os.path.exists("/dev/nvidia0"):
        pytest.skip("a GPU is visible")
    lib = _lib.load()
    h = C.c_void_p()
    rc = lib.ibmgpu_init(0, 1, 0, None, C.byref(h))
    assert rc != 0
    with pytest.raises(Exception):
        ibm.Context(0)


def test_error_codes_defined():
    txt = open(_lib.HEADER).read()
    for code in ("IBMGPU_EINVAL", "IBMGPU_ESUPPORT", "IBMGPU_ECUDA", "IBMGPU_ENCCL", "IBMGPU_ENOMEM"):
        assert code in txt
