"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU checkers.

* ``port``: the plain-C restatement (oracle/liboracle.so, source oracle/ibm_oracle.c).
* ``ref``:  the unmodified reference headers behind a C shim (oracle/_ref/libibmref.so,
  built by oracle/Makefile from /root/reference; the .so travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference leg may
import this module. The product (paper_1109_3524_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libibmref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def _d(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _i(a):
    return a.ctypes.data_as(_ip) if a is not None else None


@dataclass
class Csr:
    """Host CSR with the reference layout (sparse.hpp:214-219): int32 rp/ci, f64 values."""

    rows: int
    cols: int
    rp: np.ndarray
    ci: np.ndarray
    v: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.rp[-1])

    def dense(self) -> np.ndarray:
        d = np.zeros((self.rows, self.cols))
        for r in range(self.rows):
            d[r, self.ci[self.rp[r]:self.rp[r + 1]]] = self.v[self.rp[r]:self.rp[r + 1]]
        return d

    def diagonal(self) -> np.ndarray:
        out = np.zeros(min(self.rows, self.cols))
        for r in range(len(out)):
            seg = self.ci[self.rp[r]:self.rp[r + 1]]
            k = np.searchsorted(seg, r)
            if k < len(seg) and seg[k] == r:
                out[r] = self.v[self.rp[r] + k]
        return out

    def same_structure(self, o: "Csr") -> bool:
        return (self.rows == o.rows and self.cols == o.cols and np.array_equal(self.rp, o.rp)
                and np.array_equal(self.ci, o.ci))

    @staticmethod
    def from_dense(d: np.ndarray) -> "Csr":
        rows, cols = d.shape
        rp = np.zeros(rows + 1, np.int32)
        ci, v = [], []
        for r in range(rows):
            nz = np.nonzero(d[r])[0]
            ci.extend(nz.tolist())
            v.extend(d[r, nz].tolist())
            rp[r + 1] = len(ci)
        return Csr(rows, cols, rp, np.asarray(ci, np.int32), np.asarray(v, np.float64))

    def spmv_np(self, x: np.ndarray) -> np.ndarray:
        """Row-order accumulation in numpy (sparse.hpp:101-110), for small cases."""
        y = np.zeros(self.rows)
        for r in range(self.rows):
            s = 0.0
            for k in range(self.rp[r], self.rp[r + 1]):
                s += self.v[k] * x[self.ci[k]]
            y[r] = s
        return y


# ----------------------------------------------------------------------------- port
class _OrcCsr(C.Structure):
    _fields_ = [("rows", C.c_int), ("cols", C.c_int), ("nnz", C.c_int), ("rp", _ip), ("ci", _ip), ("v", _dp)]


class _OrcHier(C.Structure):
    _fields_ = [("n_levels", C.c_int), ("stalled", C.c_int), ("A", C.POINTER(C.POINTER(_OrcCsr))),
                ("P", C.POINTER(C.POINTER(_OrcCsr))), ("Pt", C.POINTER(C.POINTER(_OrcCsr))),
                ("inv_diag", C.POINTER(_dp)), ("omega", _dp), ("coarse_A", C.POINTER(_OrcCsr)),
                ("n_c", C.c_int), ("chol", _dp)]


class Port:
    """The C restatement (oracle/ibm_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.L = C.CDLL(path)
        P = C.POINTER(_OrcCsr)
        L.orc_csr_from.restype = P
        L.orc_csr_from.argtypes = [C.c_int, C.c_int, _ip, _ip, _dp]
        L.orc_csr_free.argtypes = [P]
        L.orc_from_triplets.restype = P
        L.orc_from_triplets.argtypes = [C.c_int, C.c_int, C.c_int, _ip, _ip, _dp]
        L.orc_spmv.argtypes = [P, _dp, _dp]
        L.orc_transpose.restype = P
        L.orc_transpose.argtypes = [P]
        L.orc_spmm_rows.restype = P
        L.orc_spmm_rows.argtypes = [P, C.c_int, C.c_int, P]
        L.orc_triple.restype = P
        L.orc_triple.argtypes = [P, P, P, C.c_int, C.POINTER(C.c_longlong), _ip]
        L.orc_add.restype = P
        L.orc_add.argtypes = [C.c_double, P, C.c_double, P]
        L.orc_symmetrized.restype = P
        L.orc_symmetrized.argtypes = [P]
        L.orc_pin.restype = P
        L.orc_pin.argtypes = [P, C.c_int]
        L.orc_concat_cols.restype = P
        L.orc_concat_cols.argtypes = [P, P]
        H = C.POINTER(_OrcHier)
        L.orc_pcg.restype = C.c_int
        L.orc_pcg.argtypes = [P, _dp, _dp, C.c_int, H, C.c_double, C.c_int, _dp, _ip, _dp, _ip, _dp, C.c_int, _ip]
        L.orc_sa_build.restype = H
        L.orc_sa_build.argtypes = [P, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int]
        L.orc_hier_free.argtypes = [H]
        L.orc_sa_apply.argtypes = [H, _dp, _dp]
        L.orc_aggregate.restype = C.c_int
        L.orc_aggregate.argtypes = [P, C.c_double, C.c_int, _ip]
        L.orc_rho.restype = C.c_double
        L.orc_rho.argtypes = [P, C.c_int]
        L.orc_delta_roma.restype = C.c_double
        L.orc_delta_roma.argtypes = [C.c_double, C.c_double]
        L.orc_assemble_EH.restype = C.c_int
        L.orc_assemble_EH.argtypes = [C.c_int, C.c_int] + [_dp] * 6 + [C.c_double, _dp, C.c_int, _dp, _dp, _dp,
                                                                       C.POINTER(P), C.POINTER(P)]

    # conversion
    def _in(self, m: Csr):
        rp = np.ascontiguousarray(m.rp, np.int32)
        ci = np.ascontiguousarray(m.ci, np.int32)
        v = np.ascontiguousarray(m.v, np.float64)
        return self.L.orc_csr_from(m.rows, m.cols, _i(rp), _i(ci if len(ci) else np.zeros(1, np.int32)),
                                   _d(v if len(v) else np.zeros(1)))

    @staticmethod
    def _out_noFree(p) -> Csr:
        s = p.contents
        rp = np.ctypeslib.as_array(s.rp, (s.rows + 1,)).copy()
        nnz = int(rp[-1])
        ci = np.ctypeslib.as_array(s.ci, (nnz,)).copy() if nnz else np.zeros(0, np.int32)
        v = np.ctypeslib.as_array(s.v, (nnz,)).copy() if nnz else np.zeros(0)
        return Csr(s.rows, s.cols, rp, ci, v)

    def _out(self, p) -> Csr:
        if not p:
            raise ValueError("oracle: invalid argument")
        m = self._out_noFree(p)
        self.L.orc_csr_free(p)
        return m

    def _with(self, *mats):
        return [self._in(m) for m in mats]

    def _free(self, ps):
        for p in ps:
            self.L.orc_csr_free(p)

    # sparse.hpp
    def from_triplets(self, rows, cols, r, c, v) -> Csr:
        r = np.ascontiguousarray(r, np.int32)
        c = np.ascontiguousarray(c, np.int32)
        v = np.ascontiguousarray(v, np.float64)
        return self._out(self.L.orc_from_triplets(rows, cols, len(r), _i(r), _i(c), _d(v)))

    def spmv(self, A: Csr, x: np.ndarray) -> np.ndarray:
        (pa,) = self._with(A)
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(A.rows)
        self.L.orc_spmv(pa, _d(x), _d(y))
        self._free([pa])
        return y

    def transpose(self, A: Csr) -> Csr:
        (pa,) = self._with(A)
        out = self._out(self.L.orc_transpose(pa))
        self._free([pa])
        return out

    def spmm(self, A: Csr, B: Csr) -> Csr:
        pa, pb = self._with(A, B)
        out = self._out(self.L.orc_spmm_rows(pa, 0, A.rows, pb))
        self._free([pa, pb])
        return out

    def triple(self, A: Csr, B: Csr, Cm: Csr, slice_rows: int):
        pa, pb, pc = self._with(A, B, Cm)
        peak = C.c_longlong(0)
        ns = C.c_int(0)
        out = self._out(self.L.orc_triple(pa, pb, pc, slice_rows, C.byref(peak), C.byref(ns)))
        self._free([pa, pb, pc])
        return out, peak.value, ns.value

    def add(self, a: float, A: Csr, b: float, B: Csr) -> Csr:
        pa, pb = self._with(A, B)
        out = self._out(self.L.orc_add(a, pa, b, pb))
        self._free([pa, pb])
        return out

    def symmetrized(self, A: Csr) -> Csr:
        (pa,) = self._with(A)
        out = self._out(self.L.orc_symmetrized(pa))
        self._free([pa])
        return out

    def pin(self, A: Csr, pin: int) -> Csr:
        (pa,) = self._with(A)
        out = self._out(self.L.orc_pin(pa, pin))
        self._free([pa])
        return out

    def concat_cols(self, G: Csr, Et: Csr) -> Csr:
        pa, pb = self._with(G, Et)
        out = self._out(self.L.orc_concat_cols(pa, pb))
        self._free([pa, pb])
        return out

    # solvers
    def sa_build(self, A: Csr, theta=0.25, max_coarse=64, max_levels=25, power_its=10, tail=0) -> "PortHier":
        (pa,) = self._with(A)
        h = self.L.orc_sa_build(pa, theta, max_coarse, max_levels, power_its, tail)
        self._free([pa])
        if not h:
            raise ValueError("oracle sa_build: invalid argument")
        return PortHier(self, h)

    def pcg(self, A: Csr, b, x0=None, kind=1, hier: "PortHier | None" = None, rel_tol=1e-5, max_iters=2000,
            history=False):
        (pa,) = self._with(A)
        b = np.ascontiguousarray(b, np.float64)
        x0a = None if x0 is None else np.ascontiguousarray(x0, np.float64)
        x = np.zeros(A.rows)
        it, st, hl = C.c_int(0), C.c_int(0), C.c_int(0)
        rr = C.c_double(0)
        hist = np.zeros(max_iters + 2) if history else None
        rc = self.L.orc_pcg(pa, _d(b), _d(x0a), kind, hier.h if hier else None, rel_tol, max_iters, _d(x),
                            C.byref(it), C.byref(rr), C.byref(st), _d(hist), len(hist) if history else 0,
                            C.byref(hl))
        self._free([pa])
        if rc:
            raise ValueError("oracle pcg: invalid argument")
        return dict(x=x, iterations=it.value, rel_residual=rr.value, status=st.value,
                    history=hist[:hl.value] if history else None)

    def aggregate(self, A: Csr, theta: float, n_core: int):
        (pa,) = self._with(A)
        agg = np.zeros(max(n_core, 1), np.int32)
        n = self.L.orc_aggregate(pa, theta, n_core, _i(agg))
        self._free([pa])
        return n, agg[:n_core]

    def rho(self, A: Csr, iters=10) -> float:
        (pa,) = self._with(A)
        r = self.L.orc_rho(pa, iters)
        self._free([pa])
        return r

    def delta_roma(self, r: float, h: float) -> float:
        return self.L.orc_delta_roma(r, h)

    def assemble_EH(self, grid: dict, px, py, ds):
        P = C.POINTER(_OrcCsr)
        E, H = P(), P()
        arr = {k: np.ascontiguousarray(grid[k], np.float64) for k in
               ("x_faces", "y_faces", "x_c", "y_c", "del_x", "del_y", "uniform")}
        px = np.ascontiguousarray(px, np.float64)
        py = np.ascontiguousarray(py, np.float64)
        ds = np.ascontiguousarray(ds, np.float64)
        rc = self.L.orc_assemble_EH(grid["nx"], grid["ny"], _d(arr["x_faces"]), _d(arr["y_faces"]), _d(arr["x_c"]),
                                    _d(arr["y_c"]), _d(arr["del_x"]), _d(arr["del_y"]), grid["h_min"],
                                    _d(arr["uniform"]), len(px), _d(px), _d(py), _d(ds), C.byref(E), C.byref(H))
        if rc:
            raise RuntimeError("body point too close to the edge of the uniform grid region")
        return self._out(E), self._out(H)


class PortHier:
    def __init__(self, port: Port, h):
        self.port, self.h = port, h

    def __del__(self):
        try:
            self.port.L.orc_hier_free(self.h)
        except Exception:
            pass

    @property
    def n_levels(self) -> int:
        return self.h.contents.n_levels

    @property
    def stalled(self) -> bool:
        return bool(self.h.contents.stalled)

    def level(self, l: int):
        s = self.h.contents
        return dict(A=Port._out_noFree(s.A[l]), P=Port._out_noFree(s.P[l]), Pt=Port._out_noFree(s.Pt[l]),
                    omega=s.omega[l])

    def coarse(self) -> Csr:
        return Port._out_noFree(self.h.contents.coarse_A)

    def apply(self, r: np.ndarray) -> np.ndarray:
        r = np.ascontiguousarray(r, np.float64)
        z = np.zeros_like(r)
        self.port.L.orc_sa_apply(self.h, _d(r), _d(z))
        return z


# ----------------------------------------------------------------------------- ref
class Ref:
    """The unmodified reference (oracle/_ref/libibmref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: build with `make -C oracle` where /root/reference exists")
        L = self.L = C.CDLL(path)
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_max_threads.restype = C.c_int
        L.ref_mat_from_csr.restype = vp
        L.ref_mat_from_csr.argtypes = [C.c_int, C.c_int, _ip, _ip, _dp]
        L.ref_mat_from_triplets.restype = vp
        L.ref_mat_from_triplets.argtypes = [C.c_int, C.c_int, C.c_int, _ip, _ip, _dp]
        L.ref_mat_free.argtypes = [vp]
        L.ref_mat_info.argtypes = [vp, _ip, _ip, _ip]
        L.ref_mat_copy.argtypes = [vp, _ip, _ip, _dp]
        L.ref_spmv.argtypes = [vp, _dp, _dp]
        for f in ("ref_transpose", "ref_symmetrized"):
            getattr(L, f).restype = vp
            getattr(L, f).argtypes = [vp]
        L.ref_spmm.restype = vp
        L.ref_spmm.argtypes = [vp, vp]
        L.ref_triple.restype = vp
        L.ref_triple.argtypes = [vp, vp, vp, C.c_int, C.POINTER(C.c_longlong), _ip]
        L.ref_add.restype = vp
        L.ref_add.argtypes = [C.c_double, vp, C.c_double, vp]
        L.ref_pin.restype = vp
        L.ref_pin.argtypes = [vp, C.c_int]
        L.ref_is_symmetric.restype = C.c_int
        L.ref_is_symmetric.argtypes = [vp, C.c_double]
        L.ref_pcg.restype = C.c_int
        L.ref_pcg.argtypes = [vp, _dp, _dp, C.c_int, vp, C.c_double, C.c_int, _dp, _ip, _dp, _ip, _dp, C.c_int, _ip]
        L.ref_sa_build.restype = vp
        L.ref_sa_build.argtypes = [vp, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_sa_free.argtypes = [vp]
        L.ref_sa_levels.restype = C.c_int
        L.ref_sa_levels.argtypes = [vp, _ip]
        L.ref_sa_level_mat.restype = vp
        L.ref_sa_level_mat.argtypes = [vp, C.c_int, C.c_int, _dp]
        L.ref_sa_apply.argtypes = [vp, _dp, C.c_int, _dp]
        L.ref_amg_solve.restype = C.c_int
        L.ref_amg_solve.argtypes = [vp, vp, _dp, C.c_double, C.c_int, _dp, _ip, _dp, _ip]
        L.ref_aggregate.restype = C.c_int
        L.ref_aggregate.argtypes = [vp, C.c_double, C.c_int, _ip]
        L.ref_strength.restype = vp
        L.ref_strength.argtypes = [vp, C.c_double, C.c_int]
        L.ref_rho.restype = C.c_double
        L.ref_rho.argtypes = [vp, C.c_int]
        L.ref_delta_roma.restype = C.c_double
        L.ref_delta_roma.argtypes = [C.c_double, C.c_double]
        L.ref_case_open.restype = vp
        L.ref_case_open.argtypes = [C.c_char_p, C.c_double, C.c_double]
        L.ref_case_free.argtypes = [vp]
        L.ref_case_dims.argtypes = [vp, _ip]
        L.ref_case_scalars.argtypes = [vp, _dp]
        L.ref_case_op.restype = vp
        L.ref_case_op.argtypes = [vp, C.c_char_p]
        L.ref_case_hier.restype = vp
        L.ref_case_hier.argtypes = [vp]
        L.ref_case_grid.restype = C.c_int
        L.ref_case_grid.argtypes = [vp, C.c_int, _dp]
        L.ref_case_uniform.argtypes = [vp, _dp]
        L.ref_case_bodies.argtypes = [vp, _dp, _dp, _dp, _dp, _dp]
        L.ref_case_step.restype = C.c_int
        L.ref_case_step.argtypes = [vp, _dp, C.c_char_p, C.c_int]
        L.ref_case_write_checkpoint.restype = C.c_int
        L.ref_case_write_checkpoint.argtypes = [vp, C.c_char_p]
        L.ref_case_read_checkpoint.restype = C.c_int
        L.ref_case_read_checkpoint.argtypes = [vp, C.c_char_p]
        L.ref_case_state.restype = C.c_int
        L.ref_case_state.argtypes = [vp, C.c_int, _dp]
        L.ref_case_time.restype = C.c_double
        L.ref_case_time.argtypes = [vp]
        L.ref_case_forces.argtypes = [vp, _dp]
        L.ref_case_boundary.restype = C.c_int
        L.ref_case_boundary.argtypes = [vp, _dp]
        L.ref_case_visc_bc.restype = C.c_int
        L.ref_case_visc_bc.argtypes = [vp, _dp]

    def err(self) -> str:
        return self.L.ref_last_error().decode()

    def set_threads(self, n: int):
        self.L.ref_set_threads(n)

    # matrices
    def _in(self, m: Csr):
        rp = np.ascontiguousarray(m.rp, np.int32)
        ci = np.ascontiguousarray(m.ci, np.int32) if m.nnz else np.zeros(1, np.int32)
        v = np.ascontiguousarray(m.v, np.float64) if m.nnz else np.zeros(1)
        return self.L.ref_mat_from_csr(m.rows, m.cols, _i(rp), _i(ci), _d(v))

    def _copy(self, p) -> Csr:
        rows, cols, nnz = C.c_int(), C.c_int(), C.c_int()
        self.L.ref_mat_info(p, C.byref(rows), C.byref(cols), C.byref(nnz))
        rp = np.zeros(rows.value + 1, np.int32)
        ci = np.zeros(max(nnz.value, 1), np.int32)
        v = np.zeros(max(nnz.value, 1))
        self.L.ref_mat_copy(p, _i(rp), _i(ci), _d(v))
        return Csr(rows.value, cols.value, rp, ci[:nnz.value], v[:nnz.value])

    def _out(self, p) -> Csr:
        if not p:
            raise ValueError(self.err())
        m = self._copy(p)
        self.L.ref_mat_free(p)
        return m

    def from_triplets(self, rows, cols, r, c, v) -> Csr:
        r = np.ascontiguousarray(r, np.int32)
        c = np.ascontiguousarray(c, np.int32)
        v = np.ascontiguousarray(v, np.float64)
        return self._out(self.L.ref_mat_from_triplets(rows, cols, len(r), _i(r), _i(c), _d(v)))

    def spmv(self, A: Csr, x) -> np.ndarray:
        p = self._in(A)
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(A.rows)
        self.L.ref_spmv(p, _d(x), _d(y))
        self.L.ref_mat_free(p)
        return y

    def _un(self, f, A: Csr, *args) -> Csr:
        p = self._in(A)
        out = self._out(f(p, *args))
        self.L.ref_mat_free(p)
        return out

    def transpose(self, A):
        return self._un(self.L.ref_transpose, A)

    def symmetrized(self, A):
        return self._un(self.L.ref_symmetrized, A)

    def pin(self, A, pin):
        return self._un(self.L.ref_pin, A, pin)

    def strength(self, A, theta, n_core):
        return self._un(self.L.ref_strength, A, theta, n_core)

    def is_symmetric(self, A, tol=1e-12) -> bool:
        p = self._in(A)
        r = self.L.ref_is_symmetric(p, tol)
        self.L.ref_mat_free(p)
        return bool(r)

    def spmm(self, A, B):
        pa, pb = self._in(A), self._in(B)
        out = self._out(self.L.ref_spmm(pa, pb))
        self.L.ref_mat_free(pa)
        self.L.ref_mat_free(pb)
        return out

    def add(self, a, A, b, B):
        pa, pb = self._in(A), self._in(B)
        out = self._out(self.L.ref_add(a, pa, b, pb))
        self.L.ref_mat_free(pa)
        self.L.ref_mat_free(pb)
        return out

    def triple(self, A, B, Cm, slice_rows):
        ps = [self._in(m) for m in (A, B, Cm)]
        peak, ns = C.c_longlong(0), C.c_int(0)
        out = self._out(self.L.ref_triple(*ps, slice_rows, C.byref(peak), C.byref(ns)))
        for p in ps:
            self.L.ref_mat_free(p)
        return out, peak.value, ns.value

    def aggregate(self, A, theta, n_core):
        p = self._in(A)
        agg = np.zeros(max(n_core, 1), np.int32)
        n = self.L.ref_aggregate(p, theta, n_core, _i(agg))
        self.L.ref_mat_free(p)
        return n, agg[:n_core]

    def rho(self, A, iters=10):
        p = self._in(A)
        r = self.L.ref_rho(p, iters)
        self.L.ref_mat_free(p)
        return r

    def delta_roma(self, r, h):
        return self.L.ref_delta_roma(r, h)

    def sa_build(self, A: Csr, theta=0.25, max_coarse=64, max_levels=25, power_its=10, tail=0) -> "RefHier":
        p = self._in(A)
        h = self.L.ref_sa_build(p, theta, max_coarse, max_levels, power_its, tail)
        self.L.ref_mat_free(p)
        if not h:
            raise ValueError(self.err())
        return RefHier(self, h, owned=True)

    def pcg(self, A: Csr, b, x0=None, kind=1, hier: "RefHier | None" = None, rel_tol=1e-5, max_iters=2000,
            history=False):
        p = self._in(A)
        b = np.ascontiguousarray(b, np.float64)
        x0a = None if x0 is None else np.ascontiguousarray(x0, np.float64)
        x = np.zeros(A.rows)
        it, st, hl = C.c_int(0), C.c_int(0), C.c_int(0)
        rr = C.c_double(0)
        hist = np.zeros(max_iters + 2) if history else None
        rc = self.L.ref_pcg(p, _d(b), _d(x0a), kind, hier.h if hier else None, rel_tol, max_iters, _d(x),
                            C.byref(it), C.byref(rr), C.byref(st), _d(hist), len(hist) if history else 0,
                            C.byref(hl))
        self.L.ref_mat_free(p)
        if rc:
            raise ValueError(self.err())
        return dict(x=x, iterations=it.value, rel_residual=rr.value, status=st.value,
                    history=hist[:hl.value] if history else None)

    def amg_solve(self, A: Csr, hier: "RefHier", b, rel_tol=1e-5, max_iters=200):
        p = self._in(A)
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(A.rows)
        it, st = C.c_int(0), C.c_int(0)
        rr = C.c_double(0)
        self.L.ref_amg_solve(p, hier.h, _d(b), rel_tol, max_iters, _d(x), C.byref(it), C.byref(rr), C.byref(st))
        self.L.ref_mat_free(p)
        return dict(x=x, iterations=it.value, rel_residual=rr.value, status=st.value)

    def case(self, cfg_path: str, h_min: float = 0.0, dt: float = 0.0) -> "RefCase":
        h = self.L.ref_case_open(cfg_path.encode(), h_min, dt)
        if not h:
            raise ValueError(self.err())
        return RefCase(self, h)


class RefHier:
    def __init__(self, ref: Ref, h, owned: bool):
        self.ref, self.h, self.owned = ref, h, owned

    def __del__(self):
        if self.owned:
            try:
                self.ref.L.ref_sa_free(self.h)
            except Exception:
                pass

    @property
    def n_levels(self) -> int:
        return self.ref.L.ref_sa_levels(self.h, None)

    @property
    def stalled(self) -> bool:
        s = C.c_int(0)
        self.ref.L.ref_sa_levels(self.h, C.byref(s))
        return bool(s.value)

    def level(self, l: int):
        om = C.c_double(0)
        A = self.ref._copy(self.ref.L.ref_sa_level_mat(self.h, l, 0, C.byref(om)))
        P = self.ref._copy(self.ref.L.ref_sa_level_mat(self.h, l, 1, None))
        Pt = self.ref._copy(self.ref.L.ref_sa_level_mat(self.h, l, 2, None))
        return dict(A=A, P=P, Pt=Pt, omega=om.value)

    def coarse(self) -> Csr:
        return self.ref._copy(self.ref.L.ref_sa_level_mat(self.h, self.n_levels, 0, None))

    def apply(self, r):
        r = np.ascontiguousarray(r, np.float64)
        z = np.zeros_like(r)
        self.ref.L.ref_sa_apply(self.h, _d(r), len(r), _d(z))
        return z


class RefCase:
    GRID = ("x_faces", "y_faces", "dx", "dy", "x_c", "y_c", "del_x", "del_y")
    STEP_KEYS = ("ok", "solve1_iters", "solve2_iters", "solve1_res", "solve2_res", "div_residual",
                 "noslip_residual", "rebuilt_hierarchy", "rebuilt_operators", "t_assembly", "t_precond",
                 "t_explicit", "t_solve1", "t_solve2", "t_projection")

    def __init__(self, ref: Ref, h):
        self.ref, self.h = ref, h
        d = np.zeros(7, np.int32)
        ref.L.ref_case_dims(h, _i(d))
        self.nx, self.ny, self.n_q, self.n_p, self.n_b, self.n_lambda, self.n_levels = map(int, d)
        s = np.zeros(5)
        ref.L.ref_case_scalars(h, _d(s))
        self.dt, self.nu, self.h_min, self.u_inf, self.ref_length = map(float, s)

    def __del__(self):
        try:
            self.ref.L.ref_case_free(self.h)
        except Exception:
            pass

    def op(self, name: str) -> Csr:
        return self.ref._copy(self.ref.L.ref_case_op(self.h, name.encode()))

    def hierarchy(self) -> RefHier:
        return RefHier(self.ref, self.ref.L.ref_case_hier(self.h), owned=False)

    def grid(self) -> dict:
        g = {"nx": self.nx, "ny": self.ny, "h_min": self.h_min}
        for i, k in enumerate(self.GRID):
            n = self.ref.L.ref_case_grid(self.h, i, None)
            a = np.zeros(n)
            self.ref.L.ref_case_grid(self.h, i, _d(a))
            g[k] = a
        u = np.zeros(4)
        self.ref.L.ref_case_uniform(self.h, _d(u))
        g["uniform"] = u
        return g

    def bodies(self) -> dict:
        out = {k: np.zeros(self.n_b) for k in ("x", "y", "ub_x", "ub_y", "ds")}
        self.ref.L.ref_case_bodies(self.h, *[_d(out[k]) for k in ("x", "y", "ub_x", "ub_y", "ds")])
        return out

    def write_checkpoint(self, path: str):
        """io.hpp:89-110 write_checkpoint of the reference Stepper."""
        if self.ref.L.ref_case_write_checkpoint(self.h, path.encode()):
            raise RuntimeError(self.ref.err())

    def read_checkpoint(self, path: str):
        """io.hpp:112-145 read_checkpoint (restores state, boundary and body positions)."""
        if self.ref.L.ref_case_read_checkpoint(self.h, path.encode()):
            raise RuntimeError(self.ref.err())

    def step(self) -> dict:
        rep = np.zeros(len(self.STEP_KEYS))
        msg = C.create_string_buffer(512)
        self.ref.L.ref_case_step(self.h, _d(rep), msg, 512)
        out = dict(zip(self.STEP_KEYS, rep.tolist()))
        out["message"] = msg.value.decode()
        return out

    def state(self, which: str) -> np.ndarray:
        k = {"q": 0, "lambda": 1, "conv_prev": 2}[which]
        n = self.ref.L.ref_case_state(self.h, k, None)
        a = np.zeros(n)
        self.ref.L.ref_case_state(self.h, k, _d(a))
        return a

    def time(self) -> float:
        return self.ref.L.ref_case_time(self.h)

    def forces(self) -> dict:
        f = np.zeros(4)
        self.ref.L.ref_case_forces(self.h, _d(f))
        return dict(fx=f[0], fy=f[1], cd=f[2], cl=f[3])

    def visc_bc(self) -> np.ndarray:
        n = self.ref.L.ref_case_visc_bc(self.h, None)
        a = np.zeros(4 * n)
        self.ref.L.ref_case_visc_bc(self.h, _d(a))
        return a

    def boundary(self) -> np.ndarray:
        n = self.ref.L.ref_case_boundary(self.h, None)
        a = np.zeros(n)
        self.ref.L.ref_case_boundary(self.h, _d(a))
        return a


_port = None
_ref = None


def port() -> Port:
    global _port
    if _port is None:
        _port = Port()
    return _port


def ref() -> Ref:
    global _ref
    if _ref is None:
        _ref = Ref()
    return _ref


def have_ref() -> bool:
    return os.path.exists(REF_SO)


# ------------------------------------------------------------------ fixtures (reference oracles.hpp)
def poisson5(n: int) -> Csr:
    """2-D five-point matrix, diag 4, neighbours -1 (proj/tests/oracles.hpp:108-120)."""
    rows, cols, vals = [], [], []
    for j in range(n):
        for i in range(n):
            p = i + j * n
            for (di, dj, v) in ((0, 0, 4.0), (-1, 0, -1.0), (1, 0, -1.0), (0, -1, -1.0), (0, 1, -1.0)):
                ii, jj = i + di, j + dj
                if 0 <= ii < n and 0 <= jj < n:
                    rows.append(p)
                    cols.append(ii + jj * n)
                    vals.append(v)
    order = np.lexsort((cols, rows))
    r = np.asarray(rows)[order]
    c = np.asarray(cols, np.int32)[order]
    v = np.asarray(vals)[order]
    rp = np.zeros(n * n + 1, np.int32)
    np.add.at(rp, r + 1, 1)
    return Csr(n * n, n * n, np.cumsum(rp).astype(np.int32), c, v)


def poisson1d(n: int) -> Csr:
    d = np.zeros((n, n))
    for i in range(n):
        d[i, i] = 2.0
        if i > 0:
            d[i, i - 1] = -1.0
        if i < n - 1:
            d[i, i + 1] = -1.0
    return Csr.from_dense(d)


def random_sparse(rows: int, cols: int, fill: float, seed: int) -> Csr:
    rng = np.random.default_rng(seed)
    mask = rng.random((rows, cols)) < fill
    d = np.where(mask, rng.uniform(-1, 1, (rows, cols)), 0.0)
    if not d.any():
        d[0, 0] = 1.0
    return Csr.from_dense(d)
