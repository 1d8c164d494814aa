"""Behavioural contracts of the reference's own unit suites, checked on the device path:
refresh policy (test_stepper.cpp:307-382), determinism (test_config.cpp:288-305), pcg(Identity)
== cg (test_krylov.cpp:113-124), V-cycle contraction and 1-D aggregation bounds
(test_krylov.cpp:143-181), stale-hierarchy robustness (:243-267), and the zero fixed point
(test_stepper.cpp:190)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1109_3524_b200 import ibm
from tests import helpers as H

pytestmark = pytest.mark.gpu


def _steps(st, n):
    out = []
    for _ in range(n):
        r = st.advance()
        assert r.ok, r.message
        out.append(r)
    return out


def test_refresh_policy_pattern_and_stationary():
    st = ibm.Stepper(H.case("flapping_smoke"), n_pc=3)
    assert [r.rebuilt_hierarchy for r in _steps(st, 7)] == [True, False, False, True, False, False, True]
    assert all(r.rebuilt_operators for r in _steps(st, 2))  # moving body: operators every step
    still = ibm.Stepper(H.case("cylinder_re40_smoke"))
    reps = _steps(still, 4)
    assert not any(r.rebuilt_hierarchy or r.rebuilt_operators for r in reps)


def test_npc1_bitwise_equals_force_rebuild():
    a = ibm.Stepper(H.case("flapping_smoke"), n_pc=1)
    b = ibm.Stepper(H.case("flapping_smoke"), force_rebuild=True)
    _steps(a, 3)
    _steps(b, 3)
    assert np.array_equal(a.get("q"), b.get("q")) and np.array_equal(a.get("lambda"), b.get("lambda"))


def test_runs_are_bitwise_deterministic():
    fa, fb = [], []
    for f, st in ((fa, ibm.Stepper(H.case("cylinder_re40_smoke"))), (fb, ibm.Stepper(H.case("cylinder_re40_smoke")))):
        for _ in range(3):
            assert st.advance().ok
            f.append(tuple(st.forces().values()))
    assert fa == fb


def test_pcg_identity_is_cg_bitwise():
    A = ibm.SparseMatrix.from_host(O.poisson5(24))
    b = np.cos(np.arange(A.rows()) * 0.11)
    p = ibm.SolverParams(record_history=True)
    r1 = ibm.cg(A, b, None, p)
    r2 = ibm.pcg(A, b, None, ibm.IdentityPreconditioner(), p)
    assert r1.iterations == r2.iterations and np.array_equal(r1.x, r2.x) and r1.history == r2.history


def test_vcycle_contraction_poisson64():
    A = O.poisson5(64)
    Ad = ibm.SparseMatrix.from_host(A)
    h = ibm.build_sa_hierarchy(Ad)
    e0 = np.random.default_rng(3).uniform(-1, 1, A.rows)
    e1 = e0 + ibm.sa_apply(h, -A.spmv_np(e0))  # one V-cycle on A e = 0
    assert np.linalg.norm(e1) <= 0.5 * np.linalg.norm(e0)


def test_poisson1d_aggregation_and_galerkin():
    A = O.poisson1d(27)
    h = ibm.build_sa_hierarchy(ibm.SparseMatrix.from_host(A), ibm.SaOptions(max_coarse=4))
    assert h.n_levels >= 1
    n_agg, _ = h.aggregates(0)
    assert 6 <= n_agg <= 13
    P = H.dev_to_csr(h.level(0)["P"]).dense()
    Ac = H.dev_to_csr(h.level(1)["A"] if h.n_levels > 1 else h.coarse_A()).dense()
    assert np.max(np.abs(Ac - P.T @ A.dense() @ P)) <= 1e-12 * np.max(np.abs(Ac))
    assert h.coarse_A().rows() <= 4


def test_stale_hierarchy_still_converges():
    st = ibm.Stepper(H.case("flapping_smoke"))
    old = ibm.SparseMatrix.from_host(H.dev_to_csr(st.op("lhs2")))
    h_old = ibm.build_sa_hierarchy(old, ibm.SaOptions(keep_fine_tail=2 * st.n_b))
    _steps(st, 2)  # the body moved: lhs2's body rows changed
    A = st.op("lhs2")
    assert not np.array_equal(H.dev_to_csr(A).v, H.dev_to_csr(old).v) or H.dev_to_csr(A).nnz != old.nnz()
    b = H.bench_rhs(A.spmv, A.rows())
    r = ibm.pcg(A, b, None, ibm.SaPreconditioner(h_old), ibm.SolverParams())
    assert r.converged() and r.rel_residual <= 1e-5


def test_zero_state_stays_bitwise_zero():
    """Quiescent cavity (no lid, no inflow): every field stays exactly zero."""
    import os
    import tempfile
    with open(H.case("cavity")) as f:
        cfg = f.read()
    cfg = "\n".join(line.replace("dirichlet 1 0", "dirichlet 0 0") for line in cfg.splitlines()) + "\n"
    with tempfile.NamedTemporaryFile("w", suffix=".cfg", delete=False) as f:
        f.write(cfg)
        path = f.name
    try:
        st = ibm.Stepper(path)
        _steps(st, 3)
        assert not np.any(st.get("q")) and not np.any(st.get("lambda"))
    finally:
        os.unlink(path)


def test_folded_tail_is_the_same_operator(monkeypatch):
    """fold.cu: the smallest levels applied as one dense operator M_l = 2W - WAW + B^T M_{l+1} B
    give the V-cycle of the unfolded hierarchy to rounding, and the same PCG iterations."""
    import bench
    cfg, h_min, dt, _ = bench.workload("c2")
    st = ibm.Stepper(H.case(cfg), h_min=h_min, dt=dt)
    A = st.op("lhs2")
    opts = ibm.SaOptions(keep_fine_tail=2 * st.n_b)
    monkeypatch.setenv("IBMGPU_FOLD", "0")
    h0 = ibm.build_sa_hierarchy(A, opts)
    monkeypatch.setenv("IBMGPU_FOLD", "1")
    h1 = ibm.build_sa_hierarchy(A, opts)
    assert h0.folded() == (0, h0.info()[2])
    nf, nd = h1.folded()
    assert nf >= 1 and nd == h1.level(h1.n_levels - nf)["A"].rows()
    assert h1.n_levels == h0.n_levels and h1.info()[2] == h0.info()[2]  # the reference structure is kept
    b = H.bench_rhs(A.spmv, A.rows())
    z0, z1 = ibm.sa_apply(h0, b), ibm.sa_apply(h1, b)
    assert np.linalg.norm(z1 - z0) <= 1e-13 * np.linalg.norm(z0)
    r0 = ibm.pcg(A, b, None, ibm.SaPreconditioner(h0), ibm.SolverParams())
    r1 = ibm.pcg(A, b, None, ibm.SaPreconditioner(h1), ibm.SolverParams())
    assert r0.iterations == r1.iterations and np.max(np.abs(r1.x - r0.x)) <= 1e-9 * np.max(np.abs(r0.x))
