"""ctypes loader for libibmgpu.so (the C-ABI in include/ibmgpu.h).

The product has no CPU fallback: if the shared library is missing or no CUDA device is
visible, every entry point raises. The library is built in-tree by `make` (or
`__graft_entry__.build()`), so the file that is loaded is the one in this directory.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
# IBMGPU_LIB: an alternative build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("IBMGPU_LIB") or os.path.join(HERE, "libibmgpu.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "ibmgpu.h")

IBMGPU_OK, IBMGPU_EINVAL, IBMGPU_ESUPPORT, IBMGPU_ECUDA, IBMGPU_ENCCL, IBMGPU_ENOMEM = range(6)

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_vp = C.c_void_p


class IbmGpuError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class SolverParamsC(C.Structure):
    _fields_ = [("rel_tol", C.c_double), ("max_iters", C.c_int), ("record_history", C.c_int),
                ("check_symmetry", C.c_int)]


class SolveResultC(C.Structure):
    _fields_ = [("iterations", C.c_int), ("rel_residual", C.c_double), ("status", C.c_int),
                ("history_len", C.c_int)]


class SaOptionsC(C.Structure):
    _fields_ = [("theta", C.c_double), ("max_coarse", C.c_int), ("max_levels", C.c_int),
                ("power_iterations", C.c_int), ("keep_fine_tail", C.c_int)]


class GridDescC(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("x_faces", _dp), ("y_faces", _dp), ("dx", _dp), ("dy", _dp),
                ("x_c", _dp), ("y_c", _dp), ("del_x", _dp), ("del_y", _dp), ("h_min", C.c_double),
                ("uniform", C.c_double * 4)]


class CaseOverridesC(C.Structure):
    _fields_ = [("h_min", C.c_double), ("dt", C.c_double), ("n_pc", C.c_int), ("force_rebuild", C.c_int),
                ("slice_rows", C.c_int)]


class EdgeBcC(C.Structure):
    _fields_ = [("kind", C.c_int), ("u", C.c_double), ("v", C.c_double)]


class BcSpecC(C.Structure):
    _fields_ = [("left", EdgeBcC), ("right", EdgeBcC), ("bottom", EdgeBcC), ("top", EdgeBcC), ("u_inf", C.c_double)]


class SolverConfigC(C.Structure):
    _fields_ = [("kind", C.c_int), ("rel_tol", C.c_double), ("max_iters", C.c_int), ("sa_theta", C.c_double),
                ("sa_max_coarse", C.c_int)]


class CaseConfigC(C.Structure):
    """ibm_case_config: the scalar part of CaseConfig (config.hpp:54-95) from the native parser."""
    _fields_ = [("domain", C.c_double * 4), ("uniform", C.c_double * 4), ("h_min", C.c_double),
                ("ratio", C.c_double * 4), ("nu", C.c_double), ("re", C.c_double), ("u_inf", C.c_double),
                ("ref_length", C.c_double), ("u0", C.c_double), ("v0", C.c_double), ("dt", C.c_double),
                ("n_steps", C.c_int), ("n_out", C.c_int), ("checkpoint_every", C.c_int), ("n_pc", C.c_int),
                ("n_order", C.c_int), ("slice_rows", C.c_int), ("n_bodies", C.c_int), ("bc", BcSpecC),
                ("solve1", SolverConfigC), ("solve2", SolverConfigC), ("out_dir", C.c_char * 512)]


class StepReportC(C.Structure):
    _fields_ = [("ok", C.c_int), ("solve1_iters", C.c_int), ("solve2_iters", C.c_int), ("solve1_res", C.c_double),
                ("solve2_res", C.c_double), ("div_residual", C.c_double), ("noslip_residual", C.c_double),
                ("rebuilt_hierarchy", C.c_int), ("rebuilt_operators", C.c_int), ("bc_cfl", C.c_double),
                ("t_assembly", C.c_double), ("t_precond", C.c_double), ("t_explicit", C.c_double),
                ("t_solve1", C.c_double), ("t_solve2", C.c_double), ("t_projection", C.c_double),
                ("message", C.c_char * 256)]


# (name, restype, argtypes) for every exported symbol
_SIGS = [
    ("ibmgpu_init", C.c_int, [C.c_int, C.c_int, C.c_int, _vp, C.POINTER(_vp)]),
    ("ibmgpu_destroy", C.c_int, [_vp]),
    ("ibmgpu_last_error", C.c_char_p, [_vp]),
    ("ibmgpu_version", C.c_char_p, []),
    ("ibmgpu_synchronize", C.c_int, [_vp]),
    ("ibmgpu_vec_alloc", C.c_int, [_vp, C.c_size_t, C.POINTER(_dp)]),
    ("ibmgpu_vec_free", C.c_int, [_vp, _dp]),
    ("ibmgpu_h2d", C.c_int, [_vp, _dp, _dp, C.c_size_t]),
    ("ibmgpu_d2h", C.c_int, [_vp, _dp, _dp, C.c_size_t]),
    ("ibmgpu_timer_start", C.c_int, [_vp]),
    ("ibmgpu_timer_stop", C.c_int, [_vp, C.POINTER(C.c_float)]),
    ("ibmgpu_launch_count", C.c_int, [_vp, C.POINTER(C.c_longlong)]),
    ("ibmgpu_csr_upload", C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _ip, _ip, _dp, C.POINTER(_vp)]),
    ("ibmgpu_csr_from_triplets", C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _ip, _ip, _dp, C.POINTER(_vp)]),
    ("ibmgpu_csr_info", C.c_int, [_vp, _ip, _ip, _ip]),
    ("ibmgpu_csr_download", C.c_int, [_vp, _vp, _ip, _ip, _dp]),
    ("ibmgpu_csr_destroy", C.c_int, [_vp, _vp]),
    ("ibmgpu_spmv", C.c_int, [_vp, _vp, _dp, _dp]),
    ("ibmgpu_spmv_host", C.c_int, [_vp, _vp, _dp, _dp]),
    ("ibmgpu_spmv_timed", C.c_int, [_vp, _vp, _dp, _dp, C.c_int, _dp]),
    ("ibmgpu_transpose", C.c_int, [_vp, _vp, C.POINTER(_vp)]),
    ("ibmgpu_spmm", C.c_int, [_vp, _vp, _vp, C.POINTER(_vp)]),
    ("ibmgpu_triple_product", C.c_int, [_vp, _vp, _vp, _vp, C.c_int, C.POINTER(_vp), C.POINTER(C.c_longlong), _ip]),
    ("ibmgpu_add", C.c_int, [_vp, C.c_double, _vp, C.c_double, _vp, C.POINTER(_vp)]),
    ("ibmgpu_symmetrized", C.c_int, [_vp, _vp, C.POINTER(_vp)]),
    ("ibmgpu_pin", C.c_int, [_vp, _vp, C.c_int, C.POINTER(_vp)]),
    ("ibmgpu_is_symmetric", C.c_int, [_vp, _vp, C.c_double, _ip]),
    ("ibmgpu_scale", C.c_int, [_vp, _vp, C.c_int, C.c_double, _dp, C.POINTER(_vp)]),
    ("ibmgpu_pcg", C.c_int, [_vp, _vp, C.c_int, _vp, _dp, _dp, C.POINTER(SolverParamsC), C.POINTER(SolveResultC), _dp]),
    ("ibmgpu_sa_build", C.c_int, [_vp, _vp, C.POINTER(SaOptionsC), C.POINTER(_vp)]),
    ("ibmgpu_sa_destroy", C.c_int, [_vp, _vp]),
    ("ibmgpu_sa_apply", C.c_int, [_vp, _vp, _dp, _dp]),
    ("ibmgpu_amg_solve", C.c_int, [_vp, _vp, _vp, _dp, _dp, C.POINTER(SolverParamsC), C.POINTER(SolveResultC)]),
    ("ibmgpu_hier_info", C.c_int, [_vp, _ip, _ip, _ip]),
    ("ibmgpu_hier_folded", C.c_int, [_vp, _ip, _ip]),
    ("ibmgpu_hier_transfers", C.c_int, [_vp, _vp, C.c_int, _ip]),
    ("ibmgpu_hier_level", C.c_int, [_vp, C.c_int, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp), _dp]),
    ("ibmgpu_hier_aggregates", C.c_int, [_vp, _vp, C.c_int, _ip, _ip]),
    ("ibmgpu_aggregate", C.c_int, [_vp, _vp, C.c_double, C.c_int, _ip, _ip]),
    ("ibmgpu_assemble_EH", C.c_int, [_vp, C.POINTER(GridDescC), C.c_int, _dp, _dp, _dp, C.POINTER(_vp), C.POINTER(_vp)]),
    ("ibmgpu_coupled_system", C.c_int, [_vp, _vp, _vp, _vp, C.c_int, C.c_int, C.POINTER(_vp), C.POINTER(_vp),
                                        C.POINTER(_vp), C.POINTER(C.c_longlong)]),
    ("ibmgpu_delta_roma", C.c_int, [_vp, C.c_int, _dp, C.c_double, _dp]),
    ("ibmgpu_stepper_create", C.c_int, [_vp, C.c_char_p, C.POINTER(CaseOverridesC), C.POINTER(_vp)]),
    ("ibmgpu_stepper_destroy", C.c_int, [_vp]),
    ("ibmgpu_stepper_dims", C.c_int, [_vp, _ip]),
    ("ibmgpu_stepper_scalars", C.c_int, [_vp, _dp]),
    ("ibmgpu_stepper_advance", C.c_int, [_vp, C.POINTER(StepReportC)]),
    ("ibmgpu_stepper_get", C.c_int, [_vp, C.c_int, _dp, _ip]),
    ("ibmgpu_stepper_set", C.c_int, [_vp, C.c_int, _dp, C.c_int]),
    ("ibmgpu_stepper_forces", C.c_int, [_vp, _dp]),
    ("ibmgpu_stepper_op", C.c_int, [_vp, C.c_char_p, C.POINTER(_vp)]),
    ("ibmgpu_stepper_hier", C.c_int, [_vp, C.POINTER(_vp)]),
    ("ibmgpu_stepper_grid", C.c_int, [_vp, C.c_int, _dp, _ip]),
    ("ibmgpu_stepper_bodies", C.c_int, [_vp, _dp, _dp, _dp, _dp, _dp]),
    ("ibmgpu_stepper_phase_ms", C.c_int, [_vp, C.POINTER(C.c_float)]),
    ("ibmgpu_stepper_vorticity", C.c_int, [_vp, _dp, _ip]),
    ("ibmgpu_hostcase_open", C.c_int, [C.c_char_p, C.POINTER(CaseOverridesC), C.POINTER(_vp), _ip, C.c_char_p, C.c_int]),
    ("ibmgpu_hostcase_array", C.c_int, [_vp, C.c_char_p, _dp, _ip]),
    ("ibmgpu_hostcase_csr", C.c_int, [_vp, C.c_char_p, _ip, _ip, _ip, _ip, _ip, _dp]),
    ("ibmgpu_hostcase_move", C.c_int, [_vp, C.c_double]),
    ("ibmgpu_hostcase_free", C.c_int, [_vp]),
    ("ibmgpu_host_case_config", C.c_int, [C.c_char_p, C.POINTER(CaseConfigC), C.c_char_p, C.c_int]),
    ("ibmgpu_csr_format_bytes", C.c_int, [_vp, _vp, C.POINTER(C.c_longlong), _ip]),
    ("ibmgpu_nccl_unique_id", C.c_int, [_vp]),
    ("ibmgpu_dist_create", C.c_int, [_vp, _vp, C.c_int, _vp, _ip, C.c_int, C.c_int, C.POINTER(_vp)]),
    ("ibmgpu_dist_info", C.c_int, [_vp, _ip]),
    ("ibmgpu_dist_pcg", C.c_int, [_vp, _dp, _dp, C.POINTER(SolverParamsC), C.POINTER(SolveResultC), _dp]),
    ("ibmgpu_dist_destroy", C.c_int, [_vp]),
    ("ibmgpu_stepper_distribute", C.c_int, [_vp, C.c_int, C.c_int]),
    ("ibmgpu_distplan_build", C.c_int, [C.c_int, C.c_int, _ip, _ip, _dp, _ip, _ip, C.c_int, C.c_int, C.POINTER(_vp)]),
    ("ibmgpu_distplan_sizes", C.c_int, [_vp, _ip]),
    ("ibmgpu_distplan_get", C.c_int, [_vp, _ip, _ip, _ip, _ip, _dp, _ip, _ip, _ip, _ip]),
    ("ibmgpu_distplan_free", C.c_int, [_vp]),
    ("ibmgpu_partition_lambda", C.c_int, [C.c_int, C.c_int, C.c_int, _ip, C.c_int, _ip]),
    ("ibmgpu_partition_coarse", C.c_int, [C.c_int, _ip, C.c_int, C.c_int, _ip, _ip]),
]

_lib = None


def header_symbols() -> list[str]:
    """Function names declared in include/ibmgpu.h."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ibmgpu_[A-Za-z0-9_]+)\s*\(", txt)))


def load() -> C.CDLL:
    """Load libibmgpu.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FileNotFoundError(f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build())")
    lib = C.CDLL(LIB_PATH)
    override = "IBMGPU_LIB" in os.environ  # A/B runs may load an older build missing newer entries
    for name, res, args in _SIGS:
        if override and not hasattr(lib, name):
            continue
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(rc: int, ctx=None):
    if rc == IBMGPU_OK:
        return
    msg = load().ibmgpu_last_error(ctx).decode(errors="replace")
    if rc == IBMGPU_EINVAL:
        raise ValueError(msg)
    raise IbmGpuError(rc, msg)
