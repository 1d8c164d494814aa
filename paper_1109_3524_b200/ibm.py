"""Python mirror of the reference's operator interface, backed by the B200 C-ABI.

Names, argument meaning and error behaviour follow /root/reference/proj/include/ibm/*.hpp
(SparseMatrix, spmm, sliced_triple_product, add_sparse, symmetrized, pin_row_col, pcg/cg with
Identity/Diagonal/SA preconditioners, build_sa_hierarchy, sa_apply, amg_solve,
assemble_interpolation/regularization, assemble_coupled_system, Stepper) so that parity tests
read like the reference's own. std::invalid_argument surfaces as ValueError and
std::runtime_error as RuntimeError (IbmGpuError). All compute runs on the GPU: there is no
CPU path in this module.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import (CaseOverridesC, GridDescC, SaOptionsC, SolveResultC, SolverParamsC, StepReportC, check, load)

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_ip)


class Context:
    """One GPU (ibmgpu_init). `Context.default()` gives a process-wide context on cuda:0."""

    _default = None

    def __init__(self, device: int = 0, nranks: int = 1, rank: int = 0, nccl_id: bytes | None = None):
        """nranks > 1: one rank of an NCCL group; nccl_id from nccl_unique_id() on rank 0 (the
        caller broadcasts it, e.g. over torch.distributed)."""
        self.lib = load()
        self.nranks, self.rank = nranks, rank
        h = C.c_void_p()
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        check(self.lib.ibmgpu_init(device, nranks, rank, idbuf, C.byref(h)))
        self.h = h

    @classmethod
    def default(cls) -> "Context":
        if cls._default is None:
            cls._default = Context(0)
        return cls._default

    def check(self, rc):
        check(rc, self.h)

    def sync(self):
        self.check(self.lib.ibmgpu_synchronize(self.h))

    def launches(self) -> int:
        n = C.c_longlong()
        self.lib.ibmgpu_launch_count(self.h, C.byref(n))
        return n.value

    def timer_start(self):
        self.check(self.lib.ibmgpu_timer_start(self.h))

    def timer_stop(self) -> float:
        ms = C.c_float()
        self.check(self.lib.ibmgpu_timer_stop(self.h, C.byref(ms)))
        return ms.value


def _ctx(ctx):
    return ctx if ctx is not None else Context.default()


class DeviceVector:
    """A device array of doubles (ibmgpu_vec_alloc)."""

    def __len__(self):
        return self.n

    def __init__(self, n: int, ctx: Context | None = None):
        self.ctx = _ctx(ctx)
        self.n = int(n)
        p = _dp()
        self.ctx.check(self.ctx.lib.ibmgpu_vec_alloc(self.ctx.h, max(self.n, 1), C.byref(p)))
        self.p = p

    @classmethod
    def from_host(cls, a, ctx: Context | None = None) -> "DeviceVector":
        a = np.ascontiguousarray(a, np.float64)
        v = cls(len(a), ctx)
        v.upload(a)
        return v

    def upload(self, a):
        a = np.ascontiguousarray(a, np.float64)
        assert len(a) == self.n
        if self.n:
            self.ctx.check(self.ctx.lib.ibmgpu_h2d(self.ctx.h, self.p, _d(a), self.n))

    def download(self) -> np.ndarray:
        out = np.zeros(self.n)
        if self.n:
            self.ctx.check(self.ctx.lib.ibmgpu_d2h(self.ctx.h, _d(out), self.p, self.n))
        return out

    def __del__(self):
        try:
            self.ctx.lib.ibmgpu_vec_free(self.ctx.h, self.p)
        except Exception:
            pass


def _as_dev(x, n: int, ctx: Context) -> DeviceVector:
    if isinstance(x, DeviceVector):
        return x
    x = np.ascontiguousarray(x if x is not None else np.zeros(n), np.float64)
    if len(x) != n:
        raise ValueError("dimension mismatch")
    return DeviceVector.from_host(x, ctx)


# ----------------------------------------------------------------------------- sparse.hpp
class SparseMatrix:
    """Device CSR (sparse.hpp:27-222). Immutable; structural ops return new matrices."""

    def __init__(self, handle, ctx: Context | None = None, owned: bool = True):
        self.ctx = _ctx(ctx)
        self.h = handle
        self.owned = owned
        r, c, n = C.c_int(), C.c_int(), C.c_int()
        self.ctx.lib.ibmgpu_csr_info(self.h, C.byref(r), C.byref(c), C.byref(n))
        self._rows, self._cols, self._nnz = r.value, c.value, n.value

    def __del__(self):
        if getattr(self, "owned", False):
            try:
                self.ctx.lib.ibmgpu_csr_destroy(self.ctx.h, self.h)
            except Exception:
                pass

    @classmethod
    def from_csr(cls, rows, cols, rp, ci, v, ctx: Context | None = None) -> "SparseMatrix":
        ctx = _ctx(ctx)
        rp = np.ascontiguousarray(rp, np.int32)
        ci = np.ascontiguousarray(ci, np.int32) if len(ci) else np.zeros(1, np.int32)
        v = np.ascontiguousarray(v, np.float64) if len(v) else np.zeros(1)
        h = C.c_void_p()
        ctx.check(ctx.lib.ibmgpu_csr_upload(ctx.h, rows, cols, int(rp[-1]), _i(rp), _i(ci), _d(v), C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def from_host(cls, m, ctx: Context | None = None) -> "SparseMatrix":
        """From any object with rows/cols/rp/ci/v (e.g. oracle.Csr)."""
        return cls.from_csr(m.rows, m.cols, m.rp, m.ci, m.v, ctx)

    @classmethod
    def from_triplets(cls, rows, cols, triplets, ctx: Context | None = None) -> "SparseMatrix":
        ctx = _ctx(ctx)
        t = list(triplets)
        r = np.asarray([x[0] for x in t] or [0], np.int32)
        c = np.asarray([x[1] for x in t] or [0], np.int32)
        v = np.asarray([x[2] for x in t] or [0.0], np.float64)
        h = C.c_void_p()
        ctx.check(ctx.lib.ibmgpu_csr_from_triplets(ctx.h, rows, cols, len(t), _i(r), _i(c), _d(v), C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def identity(cls, n, ctx=None):
        return cls.from_triplets(n, n, [(i, i, 1.0) for i in range(n)], ctx)

    @classmethod
    def diagonal(cls, d, ctx=None):
        return cls.from_triplets(len(d), len(d), [(i, i, float(x)) for i, x in enumerate(d)], ctx)

    def rows(self) -> int:
        return self._rows

    def cols(self) -> int:
        return self._cols

    def nnz(self) -> int:
        return self._nnz

    def csr(self):
        """(row_ptr, col_idx, values) on the host."""
        rp = np.zeros(self._rows + 1, np.int32)
        ci = np.zeros(max(self._nnz, 1), np.int32)
        v = np.zeros(max(self._nnz, 1))
        self.ctx.check(self.ctx.lib.ibmgpu_csr_download(self.ctx.h, self.h, _i(rp), _i(ci), _d(v)))
        return rp, ci[:self._nnz], v[:self._nnz]

    def spmv(self, x) -> np.ndarray:
        """sparse.hpp:112 — host vectors in, host vector out (H2D, device SpMV, D2H)."""
        x = np.ascontiguousarray(x, np.float64)
        if len(x) != self._cols:
            raise ValueError("spmv: dimension mismatch")
        y = np.zeros(self._rows)
        self.ctx.check(self.ctx.lib.ibmgpu_spmv_host(self.ctx.h, self.h, _d(x if len(x) else np.zeros(1)),
                                                     _d(y if len(y) else np.zeros(1))))
        return y

    def spmv_into(self, x: DeviceVector, y: DeviceVector):
        """sparse.hpp:101 — device vectors."""
        self.ctx.check(self.ctx.lib.ibmgpu_spmv(self.ctx.h, self.h, x.p, y.p))

    def _new(self, fn, *args) -> "SparseMatrix":
        h = C.c_void_p()
        self.ctx.check(fn(self.ctx.h, *args, C.byref(h)))
        return SparseMatrix(h, self.ctx)

    def format_bytes(self) -> tuple[int, int]:
        """(bytes one SpMV moves in the device format, SpMV kind) — ibmgpu_csr_format_bytes"""
        b, k = C.c_longlong(), C.c_int()
        self.ctx.check(self.ctx.lib.ibmgpu_csr_format_bytes(self.ctx.h, self.h, C.byref(b), C.byref(k)))
        return b.value, k.value

    def transpose(self) -> "SparseMatrix":
        return self._new(self.ctx.lib.ibmgpu_transpose, self.h)

    def scaled(self, a: float) -> "SparseMatrix":
        return self._new(self.ctx.lib.ibmgpu_scale, self.h, 0, a, None)

    def scaled_rows(self, d) -> "SparseMatrix":
        d = np.ascontiguousarray(d, np.float64)
        return self._new(self.ctx.lib.ibmgpu_scale, self.h, 1, 0.0, _d(d))

    def scaled_cols(self, d) -> "SparseMatrix":
        d = np.ascontiguousarray(d, np.float64)
        return self._new(self.ctx.lib.ibmgpu_scale, self.h, 2, 0.0, _d(d))


def spmm(A: SparseMatrix, B: SparseMatrix) -> SparseMatrix:
    return A._new(A.ctx.lib.ibmgpu_spmm, A.h, B.h)


@dataclass
class TripleProductStats:
    peak_slice_nnz: int = 0
    slices: int = 0


def sliced_triple_product(A, B, Cm, max_slice_rows: int, stats: TripleProductStats | None = None):
    peak, ns = C.c_longlong(), C.c_int()
    h = C.c_void_p()
    A.ctx.check(A.ctx.lib.ibmgpu_triple_product(A.ctx.h, A.h, B.h, Cm.h, max_slice_rows, C.byref(h),
                                                C.byref(peak), C.byref(ns)))
    if stats is not None:
        stats.peak_slice_nnz, stats.slices = peak.value, ns.value
    return SparseMatrix(h, A.ctx)


def add_sparse(a: float, A: SparseMatrix, b: float, B: SparseMatrix) -> SparseMatrix:
    return A._new(A.ctx.lib.ibmgpu_add, a, A.h, b, B.h)


def symmetrized(A: SparseMatrix) -> SparseMatrix:
    return A._new(A.ctx.lib.ibmgpu_symmetrized, A.h)


def pin_row_col(A: SparseMatrix, pin: int) -> SparseMatrix:
    return A._new(A.ctx.lib.ibmgpu_pin, A.h, pin)


def is_symmetric(A: SparseMatrix, tol: float) -> bool:
    r = C.c_int()
    A.ctx.check(A.ctx.lib.ibmgpu_is_symmetric(A.ctx.h, A.h, tol, C.byref(r)))
    return bool(r.value)


# ----------------------------------------------------------------------------- krylov.hpp / amg.hpp
@dataclass
class SolverParams:
    rel_tol: float = 1e-5
    max_iters: int = 2000
    record_history: bool = False
    check_symmetry: bool = False

    def validate(self):
        if not (0.0 < self.rel_tol < 1.0):
            raise ValueError("solver: rel_tol must be in (0,1)")
        if self.max_iters < 1:
            raise ValueError("solver: max_iters must be >= 1")

    def c(self):
        return SolverParamsC(self.rel_tol, self.max_iters, int(self.record_history), int(self.check_symmetry))


CONVERGED, MAX_ITERATIONS, BREAKDOWN = 0, 1, 2


@dataclass
class SolveResult:
    x: np.ndarray
    iterations: int = 0
    rel_residual: float = 0.0
    status: int = CONVERGED
    history: list = field(default_factory=list)

    def converged(self) -> bool:
        return self.status == CONVERGED


class IdentityPreconditioner:
    kind = 0
    hier = None


class DiagonalPreconditioner:
    kind = 1
    hier = None

    def __init__(self, A: SparseMatrix):
        self.A = A


@dataclass
class SaOptions:
    theta: float = 0.25
    max_coarse: int = 64
    max_levels: int = 25
    power_iterations: int = 10
    keep_fine_tail: int = 0

    def c(self):
        return SaOptionsC(self.theta, self.max_coarse, self.max_levels, self.power_iterations, self.keep_fine_tail)


class SaHierarchy:
    def __init__(self, h, ctx: Context, owned=True):
        self.h, self.ctx, self.owned = h, ctx, owned

    def __del__(self):
        if getattr(self, "owned", False):
            try:
                self.ctx.lib.ibmgpu_sa_destroy(self.ctx.h, self.h)
            except Exception:
                pass

    def info(self):
        nl, st, nc = C.c_int(), C.c_int(), C.c_int()
        self.ctx.lib.ibmgpu_hier_info(self.h, C.byref(nl), C.byref(st), C.byref(nc))
        return nl.value, bool(st.value), nc.value

    def folded(self) -> tuple[int, int]:
        """(levels folded into the dense coarse operator, its dimension) — fold.cu"""
        nf, nd = C.c_int(), C.c_int()
        self.ctx.check(self.ctx.lib.ibmgpu_hier_folded(self.h, C.byref(nf), C.byref(nd)))
        return nf.value, nd.value

    def transfers(self, mode: int = -1) -> bool:
        """Level-0 P / P^T applied through the stencil (xfer.cuh): mode 0 off, 1 on, -1 query."""
        on = C.c_int()
        self.ctx.check(self.ctx.lib.ibmgpu_hier_transfers(self.ctx.h, self.h, mode, C.byref(on)))
        return bool(on.value)

    @property
    def n_levels(self) -> int:
        return self.info()[0]

    @property
    def coarsening_stalled(self) -> bool:
        return self.info()[1]

    def level_count(self) -> int:
        return self.n_levels + 1

    def level(self, l: int) -> dict:
        A, P, Pt = C.c_void_p(), C.c_void_p(), C.c_void_p()
        om = C.c_double()
        self.ctx.check(self.ctx.lib.ibmgpu_hier_level(self.h, l, C.byref(A), C.byref(P), C.byref(Pt), C.byref(om)))
        out = dict(A=SparseMatrix(A, self.ctx, owned=False), omega=om.value)
        if P.value:
            out["P"] = SparseMatrix(P, self.ctx, owned=False)
            out["Pt"] = SparseMatrix(Pt, self.ctx, owned=False)
        return out

    def coarse_A(self) -> SparseMatrix:
        return self.level(self.n_levels)["A"]

    def aggregates(self, l: int):
        A = self.level(l)["A"]
        n = C.c_int()
        agg = np.zeros(max(A.rows(), 1), np.int32)
        self.ctx.check(self.ctx.lib.ibmgpu_hier_aggregates(self.ctx.h, self.h, l, _i(agg), C.byref(n)))
        return n.value, agg


class SaPreconditioner:
    kind = 2

    def __init__(self, h: SaHierarchy):
        self.hier = h  # non-owning, as amg.hpp:245 (keep h alive)


def build_sa_hierarchy(A: SparseMatrix, opts: SaOptions | None = None) -> SaHierarchy:
    o = (opts or SaOptions()).c()
    h = C.c_void_p()
    A.ctx.check(A.ctx.lib.ibmgpu_sa_build(A.ctx.h, A.h, C.byref(o), C.byref(h)))
    return SaHierarchy(h, A.ctx)


def sa_apply(h: SaHierarchy, r) -> np.ndarray:
    n = len(r)
    rd = _as_dev(r, n, h.ctx)
    zd = DeviceVector(n, h.ctx)
    h.ctx.check(h.ctx.lib.ibmgpu_sa_apply(h.ctx.h, h.h, rd.p, zd.p))
    return zd.download()


def pcg(A: SparseMatrix, b, x0, M, params: SolverParams) -> SolveResult:
    params.validate()
    n = A.rows()
    if A.rows() != A.cols() or len(b) != n:
        raise ValueError("pcg: dimension mismatch")
    if x0 is not None and len(x0) == 0:
        x0 = None
    bd = _as_dev(b, n, A.ctx)
    xd = _as_dev(x0, n, A.ctx)
    res = SolveResultC()
    hist = np.zeros(params.max_iters + 2) if params.record_history else None
    pc = params.c()
    A.ctx.check(A.ctx.lib.ibmgpu_pcg(A.ctx.h, A.h, M.kind, M.hier.h if M.hier is not None else None, bd.p, xd.p,
                                     C.byref(pc), C.byref(res), _d(hist) if hist is not None else None))
    return SolveResult(x=xd.download(), iterations=res.iterations, rel_residual=res.rel_residual, status=res.status,
                       history=list(hist[:res.history_len]) if hist is not None else [])


def cg(A, b, x0, params):
    return pcg(A, b, x0, IdentityPreconditioner(), params)


def amg_solve(A: SparseMatrix, h: SaHierarchy, b, x0, params: SolverParams) -> SolveResult:
    params.validate()
    n = A.rows()
    bd = _as_dev(b, n, A.ctx)
    xd = _as_dev(x0 if x0 is not None and len(x0) else None, n, A.ctx)
    res = SolveResultC()
    pc = params.c()
    A.ctx.check(A.ctx.lib.ibmgpu_amg_solve(A.ctx.h, A.h, h.h, bd.p, xd.p, C.byref(pc), C.byref(res)))
    return SolveResult(x=xd.download(), iterations=res.iterations, rel_residual=res.rel_residual, status=res.status)


# ----------------------------------------------------------------------------- operators.hpp
def grid_desc(g: dict) -> tuple:
    """ibm_grid_desc from a dict of grid arrays (keeps the numpy arrays alive)."""
    keep = {k: np.ascontiguousarray(g[k], np.float64) for k in
            ("x_faces", "y_faces", "dx", "dy", "x_c", "y_c", "del_x", "del_y")}
    d = GridDescC(g["nx"], g["ny"], *[_d(keep[k]) for k in
                                      ("x_faces", "y_faces", "dx", "dy", "x_c", "y_c", "del_x", "del_y")],
                  g["h_min"], (C.c_double * 4)(*[float(u) for u in g["uniform"]]))
    return d, keep


def assemble_interpolation_regularization(grid: dict, px, py, ds, ctx: Context | None = None):
    """(E, H) = assemble_interpolation / assemble_regularization (operators.hpp:264-342)."""
    ctx = _ctx(ctx)
    d, keep = grid_desc(grid)
    px = np.ascontiguousarray(px, np.float64)
    py = np.ascontiguousarray(py, np.float64)
    ds = np.ascontiguousarray(ds, np.float64)
    E, H = C.c_void_p(), C.c_void_p()
    z = np.zeros(1)
    ctx.check(ctx.lib.ibmgpu_assemble_EH(ctx.h, C.byref(d), len(px), _d(px if len(px) else z), _d(py if len(py) else z),
                                         _d(ds if len(ds) else z), C.byref(E), C.byref(H)))
    return SparseMatrix(E, ctx), SparseMatrix(H, ctx)


def assemble_coupled_system(G: SparseMatrix, E: SparseMatrix, BN: SparseMatrix, pin: int, slice_rows: int,
                            stats: TripleProductStats | None = None):
    """(Q, QT, lhs2) = assemble_coupled_system (operators.hpp:408-417)."""
    Q, QT, L2 = C.c_void_p(), C.c_void_p(), C.c_void_p()
    peak = C.c_longlong()
    G.ctx.check(G.ctx.lib.ibmgpu_coupled_system(G.ctx.h, G.h, E.h, BN.h, pin, slice_rows, C.byref(Q), C.byref(QT),
                                                C.byref(L2), C.byref(peak)))
    if stats is not None:
        stats.peak_slice_nnz = peak.value
    return SparseMatrix(Q, G.ctx), SparseMatrix(QT, G.ctx), SparseMatrix(L2, G.ctx)


def delta_roma(r, h: float, ctx: Context | None = None) -> np.ndarray:
    ctx = _ctx(ctx)
    r = np.ascontiguousarray(np.atleast_1d(r), np.float64)
    out = np.zeros_like(r)
    ctx.check(ctx.lib.ibmgpu_delta_roma(ctx.h, len(r), _d(r), h, _d(out)))
    return out


# ----------------------------------------------------------------------------- stepper.hpp
@dataclass
class StepReport:
    ok: bool
    message: str
    solve1_iters: int
    solve2_iters: int
    solve1_res: float
    solve2_res: float
    div_residual: float
    noslip_residual: float
    rebuilt_hierarchy: bool
    rebuilt_operators: bool
    bc_cfl: float
    t_assembly: float
    t_precond: float
    t_explicit: float
    t_solve1: float
    t_solve2: float
    t_projection: float


class Stepper:
    """Device-resident Stepper (stepper.hpp:169-370) over a case file (config.hpp format)."""

    STATE = {"q": 0, "lambda": 1, "conv_prev": 2, "boundary": 3, "scalars": 4, "f_tilde": 5}
    GRID = ("x_faces", "y_faces", "dx", "dy", "x_c", "y_c", "del_x", "del_y")

    def __init__(self, cfg_path: str, h_min: float = 0.0, dt: float = 0.0, n_pc: int = 0,
                 force_rebuild: bool = False, slice_rows: int = 0, ctx: Context | None = None):
        self.ctx = _ctx(ctx)
        ov = CaseOverridesC(h_min, dt, n_pc, int(force_rebuild), slice_rows)
        h = C.c_void_p()
        self.ctx.check(self.ctx.lib.ibmgpu_stepper_create(self.ctx.h, cfg_path.encode(), C.byref(ov), C.byref(h)))
        self.h = h
        d = np.zeros(8, np.int32)
        self.ctx.check(self.ctx.lib.ibmgpu_stepper_dims(self.h, _i(d)))
        (self.nx, self.ny, self.n_q, self.n_p, self.n_b, self.n_lambda, self.n_levels, self.nnz_lhs2) = map(int, d)

    def __del__(self):
        try:
            self.ctx.lib.ibmgpu_stepper_destroy(self.h)
        except Exception:
            pass

    def scalars(self) -> dict:
        s = np.zeros(6)
        self.ctx.check(self.ctx.lib.ibmgpu_stepper_scalars(self.h, _d(s)))
        return dict(zip(("dt", "nu", "h_min", "u_inf", "ref_length", "t"), s.tolist()))

    def advance(self) -> StepReport:
        r = StepReportC()
        self.ctx.check(self.ctx.lib.ibmgpu_stepper_advance(self.h, C.byref(r)))
        return StepReport(bool(r.ok), r.message.decode(errors="replace"), r.solve1_iters, r.solve2_iters,
                          r.solve1_res, r.solve2_res, r.div_residual, r.noslip_residual, bool(r.rebuilt_hierarchy),
                          bool(r.rebuilt_operators), r.bc_cfl, r.t_assembly, r.t_precond, r.t_explicit, r.t_solve1,
                          r.t_solve2, r.t_projection)

    def get(self, which: str) -> np.ndarray:
        n = C.c_int()
        k = self.STATE[which]
        self.ctx.check(self.ctx.lib.ibmgpu_stepper_get(self.h, k, None, C.byref(n)))
        out = np.zeros(max(n.value, 1))
        self.ctx.check(self.ctx.lib.ibmgpu_stepper_get(self.h, k, _d(out), C.byref(n)))
        return out[:n.value]

    def set(self, which: str, a):
        a = np.ascontiguousarray(a, np.float64)
        self.ctx.check(self.ctx.lib.ibmgpu_stepper_set(self.h, self.STATE[which], _d(a), len(a)))

    def forces(self) -> dict:
        f = np.zeros(4)
        self.ctx.check(self.ctx.lib.ibmgpu_stepper_forces(self.h, _d(f)))
        return dict(fx=f[0], fy=f[1], cd=f[2], cl=f[3])

    def op(self, name: str) -> SparseMatrix:
        h = C.c_void_p()
        self.ctx.check(self.ctx.lib.ibmgpu_stepper_op(self.h, name.encode(), C.byref(h)))
        return SparseMatrix(h, self.ctx, owned=False)

    def hierarchy(self) -> SaHierarchy:
        h = C.c_void_p()
        self.ctx.check(self.ctx.lib.ibmgpu_stepper_hier(self.h, C.byref(h)))
        return SaHierarchy(h, self.ctx, owned=False)

    def grid(self) -> dict:
        g = {"nx": self.nx, "ny": self.ny}
        for i, k in enumerate(self.GRID):
            n = C.c_int()
            self.ctx.check(self.ctx.lib.ibmgpu_stepper_grid(self.h, i, None, C.byref(n)))
            a = np.zeros(n.value)
            self.ctx.check(self.ctx.lib.ibmgpu_stepper_grid(self.h, i, _d(a), C.byref(n)))
            g[k] = a
        return g

    def bodies(self) -> dict:
        out = {k: np.zeros(max(self.n_b, 1)) for k in ("x", "y", "ub_x", "ub_y", "ds")}
        self.ctx.check(self.ctx.lib.ibmgpu_stepper_bodies(self.h, *[_d(out[k]) for k in
                                                                    ("x", "y", "ub_x", "ub_y", "ds")]))
        return {k: v[:self.n_b] for k, v in out.items()}

    _CKPT_BOUNDARY = ("left_u", "right_u", "left_v", "right_v", "bottom_v", "top_v", "bottom_u", "top_u")

    def _boundary_sizes(self):
        nx, ny = self.nx, self.ny
        return (ny, ny, ny - 1, ny - 1, nx, nx, nx - 1, nx - 1)

    def write_checkpoint(self, path: str):
        """write_checkpoint (io.hpp:89-110): the reference's 'ibmcfd-checkpoint 1' text format,
        every double as %.17g (exact round trip), readable by the reference's read_checkpoint."""
        t, step, have = self.get("scalars")

        def block(f, name, a):
            f.write(f"{name} {len(a)}\n")
            if len(a):
                np.savetxt(f, np.asarray(a, np.float64), fmt="%.17g")

        with open(path, "w") as f:
            f.write("ibmcfd-checkpoint 1\n")
            f.write("t %.17g\n" % t)
            f.write("step %d\n" % int(step))
            f.write("have_conv %d\n" % (1 if have else 0))
            block(f, "q", self.get("q"))
            block(f, "conv_prev", self.get("conv_prev"))
            block(f, "lambda", self.get("lambda"))
            bnd = self.get("boundary")
            o = 0
            for name, n in zip(self._CKPT_BOUNDARY, self._boundary_sizes()):
                block(f, name, bnd[o:o + n])
                o += n

    def read_checkpoint(self, path: str):
        """read_checkpoint (io.hpp:112-145): restores t, step, have_conv, q, conv_prev, lambda and
        the boundary arrays; body positions follow the restored time (sync_bodies_to_time)."""
        with open(path) as f:
            tok = f.read().split()
        pos = 0

        def take(n=1):
            nonlocal pos
            out = tok[pos:pos + n]
            pos += n
            return out

        magic, ver = take(2)
        if magic != "ibmcfd-checkpoint" or ver != "1":
            raise RuntimeError(f"checkpoint: bad header in {path}")
        vals = {}
        for key in ("t", "step", "have_conv"):
            k, v = take(2)
            if k != key:
                raise RuntimeError(f"checkpoint: missing {key}")
            vals[key] = float(v)
        blocks = {}
        for name in ("q", "conv_prev", "lambda") + self._CKPT_BOUNDARY:
            k, n = take(2)
            if k != name:
                raise RuntimeError(f"checkpoint: expected block '{name}', found '{k}'")
            blocks[name] = np.array([float(x) for x in take(int(n))], np.float64)
        if len(blocks["q"]) != self.n_q:
            raise RuntimeError("checkpoint: grid size mismatch")
        self.set("q", blocks["q"])
        self.set("conv_prev", blocks["conv_prev"])
        self.set("lambda", blocks["lambda"])
        self.set("boundary", np.concatenate([blocks[n] for n in self._CKPT_BOUNDARY]))
        self.set("scalars", np.array([vals["t"], vals["step"], vals["have_conv"]]))

    def vorticity(self) -> np.ndarray:
        """compute_vorticity (diagnostics.hpp:42-56) of the current q, on the device."""
        n = C.c_int()
        self.ctx.check(self.ctx.lib.ibmgpu_stepper_vorticity(self.h, None, C.byref(n)))
        w = np.zeros(max(n.value, 1))
        self.ctx.check(self.ctx.lib.ibmgpu_stepper_vorticity(self.h, _d(w), C.byref(n)))
        return w[:n.value]

    def distribute(self, virtual_ranks: int = 0, min_dist_rows: int = 200000):
        """Row-slab solve 2 (ibmgpu_stepper_distribute): over the context's NCCL ranks, or
        `virtual_ranks` emulated ranks on this GPU (0: back to the single-GPU solve)."""
        self.ctx.check(self.ctx.lib.ibmgpu_stepper_distribute(self.h, virtual_ranks, min_dist_rows))

    def phase_ms(self) -> dict:
        a = (C.c_float * 6)()
        self.ctx.check(self.ctx.lib.ibmgpu_stepper_phase_ms(self.h, a))
        return dict(zip(("assembly", "precond", "explicit", "solve1", "solve2", "projection"), list(a)))


class HostCase:
    """Host half of case loading (no GPU): grid, bodies, M, L, G exactly as the product builds them."""

    def __init__(self, cfg_path: str, h_min: float = 0.0, dt: float = 0.0):
        self.lib = load()
        ov = CaseOverridesC(h_min, dt, 0, 0, 0)
        h = C.c_void_p()
        d = np.zeros(8, np.int32)
        err = C.create_string_buffer(512)
        rc = self.lib.ibmgpu_hostcase_open(cfg_path.encode(), C.byref(ov), C.byref(h), _i(d), err, 512)
        if rc == 1:
            raise ValueError(err.value.decode())
        if rc:
            raise RuntimeError(err.value.decode())
        self.h = h
        (self.nx, self.ny, self.n_q, self.n_p, self.n_b, self.n_lambda) = map(int, d[:6])

    def __del__(self):
        try:
            self.lib.ibmgpu_hostcase_free(self.h)
        except Exception:
            pass

    def array(self, name: str) -> np.ndarray:
        n = C.c_int()
        if self.lib.ibmgpu_hostcase_array(self.h, name.encode(), None, C.byref(n)):
            raise ValueError(name)
        out = np.zeros(max(n.value, 1))
        self.lib.ibmgpu_hostcase_array(self.h, name.encode(), _d(out), C.byref(n))
        return out[:n.value]

    def csr(self, name: str):
        r, c, n = C.c_int(), C.c_int(), C.c_int()
        if self.lib.ibmgpu_hostcase_csr(self.h, name.encode(), C.byref(r), C.byref(c), C.byref(n), None, None, None):
            raise ValueError(name)
        rp = np.zeros(r.value + 1, np.int32)
        ci = np.zeros(max(n.value, 1), np.int32)
        v = np.zeros(max(n.value, 1))
        self.lib.ibmgpu_hostcase_csr(self.h, name.encode(), None, None, None, _i(rp), _i(ci), _d(v))
        return r.value, c.value, rp, ci[:n.value], v[:n.value]

    def move(self, t: float):
        self.lib.ibmgpu_hostcase_move(self.h, t)


# ----------------------------------------------------------------------------- row-slab multi-GPU (§8(e))
def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it; broadcast it to the other ranks)."""
    buf = C.create_string_buffer(128)
    check(load().ibmgpu_nccl_unique_id(buf))
    return buf.raw


def partition_lambda(nx: int, ny: int, body_cell_j, nranks: int) -> np.ndarray:
    """Row owners of the coupled system: pressure rows by balanced j-slabs, the force rows of body
    point k by the slab containing cell row body_cell_j[k] (host only)."""
    bj = np.ascontiguousarray(body_cell_j, np.int32)
    out = np.zeros(nx * ny + 2 * len(bj), np.int32)
    check(load().ibmgpu_partition_lambda(nx, ny, len(bj), _i(bj), nranks, _i(out)))
    return out


def partition_coarse(agg, n_core: int, n_agg: int, tail: int, owner_fine) -> np.ndarray:
    """Owners of the next coarser level: aggregate -> owner of its lowest-index member; the
    identity tail keeps its owners (host only)."""
    a = np.ascontiguousarray(np.asarray(agg)[:n_core], np.int32)
    of = np.ascontiguousarray(owner_fine, np.int32)
    out = np.zeros(n_agg + tail, np.int32)
    check(load().ibmgpu_partition_coarse(n_core, _i(a), n_agg, tail, _i(of), _i(out)))
    return out


def block_partition(n: int, nranks: int) -> np.ndarray:
    """Contiguous balanced row blocks."""
    return ((np.arange(n, dtype=np.int64) * nranks) // max(n, 1)).astype(np.int32)


@dataclass
class DistPlan:
    """One rank's part of a CSR matrix under row/column owners (host-only halo planning)."""
    rows: np.ndarray
    own: np.ndarray
    rptr: np.ndarray
    cidx: np.ndarray
    val: np.ndarray
    recv_off: np.ndarray
    halo: np.ndarray
    send_off: np.ndarray
    send_idx: np.ndarray

    @staticmethod
    def build(rows, cols, rptr, cidx, val, row_owner, col_owner, rank, nranks) -> "DistPlan":
        lib = load()
        rp, ci = np.ascontiguousarray(rptr, np.int32), np.ascontiguousarray(cidx, np.int32)
        v = np.ascontiguousarray(val, np.float64)
        ro, co = np.ascontiguousarray(row_owner, np.int32), np.ascontiguousarray(col_owner, np.int32)
        h = C.c_void_p()
        check(lib.ibmgpu_distplan_build(rows, cols, _i(rp), _i(ci), _d(v), _i(ro), _i(co), rank, nranks, C.byref(h)))
        try:
            sz = np.zeros(6, np.int32)
            lib.ibmgpu_distplan_sizes(h, _i(sz))
            nrow, nown, nhalo, nnz, nsend, R = (int(x) for x in sz)
            out = DistPlan(np.zeros(max(nrow, 1), np.int32), np.zeros(max(nown, 1), np.int32),
                           np.zeros(nrow + 1, np.int32), np.zeros(max(nnz, 1), np.int32), np.zeros(max(nnz, 1)),
                           np.zeros(R + 1, np.int32), np.zeros(max(nhalo, 1), np.int32), np.zeros(R + 1, np.int32),
                           np.zeros(max(nsend, 1), np.int32))
            lib.ibmgpu_distplan_get(h, _i(out.rows), _i(out.own), _i(out.rptr), _i(out.cidx), _d(out.val),
                                    _i(out.recv_off), _i(out.halo), _i(out.send_off), _i(out.send_idx))
            out.rows, out.own, out.halo = out.rows[:nrow], out.own[:nown], out.halo[:nhalo]
            out.cidx, out.val, out.send_idx = out.cidx[:nnz], out.val[:nnz], out.send_idx[:nsend]
            return out
        finally:
            lib.ibmgpu_distplan_free(h)


class DistSolver:
    """Row-slab distributed PCG (ibmgpu_dist_*): the distributed form of pcg(A, b, x0, M) with M
    identity, diagonal or SA. A and the hierarchy are the full operators; `owner` gives each row's
    rank. With a single-rank context, `virtual_ranks` > 1 emulates the partition on this GPU."""

    def __init__(self, A: SparseMatrix, M, owner, virtual_ranks: int = 1, min_dist_rows: int = 0):
        self.ctx, self.A, self.M = A.ctx, A, M
        own = np.ascontiguousarray(owner, np.int32)
        if len(own) != A.rows():
            raise ValueError("dist: owner length must equal the matrix rows")
        h = C.c_void_p()
        self.ctx.check(self.ctx.lib.ibmgpu_dist_create(self.ctx.h, A.h, M.kind, M.hier.h if M.hier is not None else None,
                                                       _i(own), virtual_ranks, min_dist_rows, C.byref(h)))
        self.h = h

    def info(self) -> dict:
        a = np.zeros(8, np.int32)
        self.ctx.lib.ibmgpu_dist_info(self.h, _i(a))
        keys = ("nranks", "dist_levels", "loopback", "own_rows", "halo", "local_ranks", "levels", "spmv_kind")
        return dict(zip(keys, (int(x) for x in a)))

    def solve(self, b, x0=None, params: SolverParams | None = None) -> SolveResult:
        params = params or SolverParams()
        params.validate()
        n = self.A.rows()
        bd = _as_dev(b, n, self.ctx)
        xd = _as_dev(x0 if x0 is not None and len(x0) else None, n, self.ctx)
        res = SolveResultC()
        hist = np.zeros(params.max_iters + 2) if params.record_history else None
        pc = params.c()
        self.ctx.check(self.ctx.lib.ibmgpu_dist_pcg(self.h, bd.p, xd.p, C.byref(pc), C.byref(res),
                                                    _d(hist) if hist is not None else None))
        return SolveResult(x=xd.download(), iterations=res.iterations, rel_residual=res.rel_residual,
                           status=res.status, history=list(hist[:res.history_len]) if hist is not None else [])

    def __del__(self):
        try:
            self.ctx.lib.ibmgpu_dist_destroy(self.h)
        except Exception:
            pass


# ----------------------------------------------------------------------------- run loop (runner.hpp)
def case_config(cfg_path: str):
    """parse_config (config.hpp:236-355) by the library's native parser: the scalar CaseConfig
    fields (n_steps, n_out, out_dir, checkpoint_every, ...) exactly as the reference reads them."""
    from ._lib import IBMGPU_EINVAL, CaseConfigC
    cfg = CaseConfigC()
    err = C.create_string_buffer(512)
    rc = load().ibmgpu_host_case_config(cfg_path.encode(), C.byref(cfg), err, 512)
    if rc:
        msg = err.value.decode(errors="replace")
        raise ValueError(msg) if rc == IBMGPU_EINVAL else RuntimeError(msg)
    return cfg


@dataclass
class RunResult:
    """runner.hpp:44-55 RunResult (the fields a caller reads)."""
    exit_code: int = 0
    message: str = ""
    steps_done: int = 0
    total_solve1_iters: int = 0
    total_solve2_iters: int = 0
    hierarchy_builds: int = 1
    max_div_residual: float = 0.0
    max_noslip_residual: float = 0.0
    force_t: list = field(default_factory=list)
    force_cd: list = field(default_factory=list)
    force_cl: list = field(default_factory=list)


def run_case(cfg_path: str, out_dir: str | None = None, n_steps: int = 0, resume_from: str = "",
             quiet: bool = True, **stepper_kw) -> RunResult:
    """run_case (runner.hpp:77-164) on the device stepper, with the reference's output files:
    forces.csv ("t,fx,fy,cd,cl", %.17g), vorticity_<k>.txt every n_out steps and at the end
    ("x y omega", %.9g), checkpoint_<k>.txt every checkpoint_every steps and checkpoint_final.txt
    (io.hpp format)."""
    import os
    cfg = case_config(cfg_path)
    out = out_dir or cfg.out_dir.decode()
    os.makedirs(out, exist_ok=True)
    n_total = n_steps or cfg.n_steps
    n_out = cfg.n_out
    ckpt_every = cfg.checkpoint_every
    st = Stepper(cfg_path, **stepper_kw)
    if resume_from:
        st.read_checkpoint(resume_from)
    g = st.grid()
    res = RunResult()
    start = int(st.get("scalars")[1])
    last_ckpt = ""

    def vort(path):
        w = st.vorticity()
        xs, ys = g["x_faces"][1:st.nx], g["y_faces"][1:st.ny]
        X, Y = np.meshgrid(xs, ys)
        with open(path, "w") as f:
            f.write(f"# vorticity at interior vertices: x y omega ({st.nx - 1} x {st.ny - 1})\n")
            np.savetxt(f, np.column_stack([X.ravel(), Y.ravel(), w]), fmt="%.9g")

    with open(os.path.join(out, "forces.csv"), "w") as fw:
        fw.write("t,fx,fy,cd,cl\n")
        for k in range(start, n_total):
            rep = st.advance()
            res.total_solve1_iters += rep.solve1_iters
            res.total_solve2_iters += rep.solve2_iters
            res.hierarchy_builds += int(rep.rebuilt_hierarchy)
            res.max_div_residual = max(res.max_div_residual, rep.div_residual)
            res.max_noslip_residual = max(res.max_noslip_residual, rep.noslip_residual)
            if not rep.ok:
                res.exit_code = 1
                res.message = rep.message + (f"; last good checkpoint: {last_ckpt}" if last_ckpt else "")
                return res
            if st.n_b > 0:
                f = st.forces()
                t = float(st.get("scalars")[0])
                fw.write("%.17g,%.17g,%.17g,%.17g,%.17g\n" % (t, f["fx"], f["fy"], f["cd"], f["cl"]))
                fw.flush()
                res.force_t.append(t)
                res.force_cd.append(f["cd"])
                res.force_cl.append(f["cl"])
            if n_out > 0 and (k + 1) % n_out == 0:
                vort(os.path.join(out, f"vorticity_{k + 1}.txt"))
            if ckpt_every > 0 and (k + 1) % ckpt_every == 0:
                last_ckpt = os.path.join(out, f"checkpoint_{k + 1}.txt")
                st.write_checkpoint(last_ckpt)
            res.steps_done = k + 1
            if not quiet and ((k + 1) % 100 == 0 or k + 1 == n_total):
                print(f"step {k + 1:6d}/{n_total}  s1 {rep.solve1_iters:3d}  s2 {rep.solve2_iters:3d}  "
                      f"div {rep.div_residual:.2e}  slip {rep.noslip_residual:.2e}")
    vort(os.path.join(out, "vorticity_final.txt"))
    st.write_checkpoint(os.path.join(out, "checkpoint_final.txt"))
    return res
