"""Level-0 grid transfers applied through the pressure stencil (csrc/xfer.cuh) instead of the
explicit P / P^T of amg.hpp:163-183.

The operator is the reference's; only the rounding differs (P's entries are not formed). The
tests pin (1) the algebra — the implicit P^T r and P e equal the explicit products of the
device-built (reference-exact) P / P^T, computed here in numpy from the downloaded level; (2) the
kernels — the V-cycle with the transfers agrees with the explicit-P V-cycle to ~1e-15 and stays
linear, self-adjoint and run-to-run deterministic; (3) the contract — PCG iteration counts
within +-2 (here equal) and solutions within 1e-6; (4) eligibility — matrices that are not a
single-stride band with tail-column extras keep the explicit path."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import oracle as O
from paper_1109_3524_b200 import ibm
from tests import helpers as H

pytestmark = pytest.mark.gpu


def _scipy(m):
    rp, ci, v = m.csr()
    return sp.csr_matrix((v, ci, rp), shape=(m.rows(), m.cols()))


@pytest.fixture(scope="module", params=["cylinder_re40_smoke", "flapping_smoke"])
def case_hier(request):
    st = ibm.Stepper(H.case(request.param))
    return request.param, st, st.hierarchy()


def test_level0_transfers_active_on_stepper_cases(case_hier):
    _, _, hh = case_hier
    assert hh.transfers() is True


def test_implicit_transfer_algebra_matches_explicit_p(case_hier):
    """(P^T r)_a = t_a sum_{m in a} [r_m - sum_{i core} A_im wd_i r_i], (P e)_k = y_k - wd_k (A y)_k
    with y = T e, and the identity on the body tail (xfer.cuh header)."""
    _, _, hh = case_hier
    lv = hh.level(0)
    A, P, Pt = _scipy(lv["A"]), _scipy(lv["P"]), _scipy(lv["Pt"])
    n = A.shape[0]
    n_agg, agg = hh.aggregates(0)
    n_core = n - (P.shape[1] - n_agg)
    agg = agg[:n_core]
    size = np.bincount(agg, minlength=n_agg)
    t = 1.0 / np.sqrt(size.astype(float))
    wd = lv["omega"] / A.diagonal()
    T = sp.csr_matrix((t[agg], agg, np.arange(n_core + 1)), shape=(n_core, n_agg))
    rng = np.random.default_rng(7)
    r, e = rng.uniform(-1, 1, n), rng.uniform(-1, 1, P.shape[1])
    u = wd * r
    u[n_core:] = 0.0
    s = r[:n_core] - (A.T @ u)[:n_core]
    rc = np.concatenate([T.T @ s, r[n_core:]])
    ref = Pt @ r
    assert np.max(np.abs(rc - ref)) <= 1e-13 * np.max(np.abs(ref))
    y = np.zeros(n)
    y[:n_core] = T @ e[:n_agg]
    pe = np.concatenate([(y - wd * (A @ y))[:n_core], e[n_agg:]])
    ref = P @ e
    assert np.max(np.abs(pe - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_vcycle_with_transfers_matches_explicit_and_is_deterministic(case_hier):
    _, _, hh = case_hier
    n = hh.level(0)["A"].rows()
    rng = np.random.default_rng(11)
    r1, r2 = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    assert hh.transfers(1)
    z1, z2, zs = ibm.sa_apply(hh, r1), ibm.sa_apply(hh, r2), ibm.sa_apply(hh, r1 + r2)
    assert np.array_equal(ibm.sa_apply(hh, r1), z1)  # fixed summation order
    assert np.max(np.abs(zs - z1 - z2)) <= 1e-12 * np.linalg.norm(zs)
    assert abs(z1 @ r2 - r1 @ z2) <= 1e-12 * abs(r1 @ z2)
    assert not hh.transfers(0)
    z1e = ibm.sa_apply(hh, r1)
    assert hh.transfers(1)
    assert np.max(np.abs(z1 - z1e)) <= 1e-13 * np.max(np.abs(z1e))


def test_pcg_with_transfers_within_contract(case_hier):
    _, _, hh = case_hier
    A = hh.level(0)["A"]
    b = np.random.default_rng(5).uniform(-1, 1, A.rows())
    p = ibm.SolverParams(rel_tol=1e-8)
    hh.transfers(0)
    r0 = ibm.pcg(A, b, None, ibm.SaPreconditioner(hh), p)
    hh.transfers(1)
    r1 = ibm.pcg(A, b, None, ibm.SaPreconditioner(hh), p)
    assert r0.converged() and r1.converged()
    assert abs(r1.iterations - r0.iterations) <= 2
    assert np.max(np.abs(r1.x - r0.x)) <= 1e-6 * np.max(np.abs(r0.x))


def test_poisson_without_tail_uses_transfers():
    A = ibm.SparseMatrix.from_host(O.poisson5(96))
    h = ibm.build_sa_hierarchy(A)
    assert h.transfers()
    b = np.random.default_rng(2).uniform(-1, 1, A.rows())
    z = ibm.sa_apply(h, b)
    h.transfers(0)
    ze = ibm.sa_apply(h, b)
    assert np.max(np.abs(z - ze)) <= 1e-13 * np.max(np.abs(ze))


def test_ineligible_matrices_keep_explicit_transfers():
    # not a stencil (random pattern) and too small for the band plan
    M = O.random_sparse(300, 300, 0.05, 3)
    S = sp.csr_matrix((M.v, M.ci, M.rp), shape=(300, 300))
    S = S + S.T + sp.eye(300) * 40.0
    S = S.tocsr()
    A = ibm.SparseMatrix.from_csr(300, 300, S.indptr, S.indices, S.data)
    h = ibm.build_sa_hierarchy(A)
    assert h.transfers(1) is False
    assert ibm.sa_apply(h, np.ones(300)).shape == (300,)


_C16_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from oracle import oracle as O
from paper_1109_3524_b200 import ibm
A = ibm.SparseMatrix.from_host(O.poisson5(320))
h = ibm.build_sa_hierarchy(A)
out, kinds = {}, []
rng = np.random.default_rng(4)
for l in range(h.n_levels):
    lv = h.level(l)
    for k in ("A", "P", "Pt"):
        m = lv[k]
        out["%s%d" % (k, l)] = m.spmv(rng.uniform(-1, 1, m.cols()))
        kinds.append(m.format_bytes()[1])
np.savez(sys.argv[2], kinds=np.array(kinds), **out)
"""


def test_sixteen_bit_column_codes_are_bitwise(tmp_path):
    """IBMGPU_C16=1 (off by default since the level-0 transfers): the SELL kernels over 16-bit
    column codes give the same bits as over int32 columns, on every SA level of a 102k-row
    Poisson hierarchy."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for flag in ("0", "1"):
        f = tmp_path / ("c16_%s.npz" % flag)
        env = dict(os.environ, IBMGPU_C16=flag)
        r = subprocess.run([sys.executable, "-c", _C16_SCRIPT, root, str(f)], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[flag] = np.load(f)
    assert any(k & 16 for k in res["1"]["kinds"]) and not any(k & 16 for k in res["0"]["kinds"])
    for k in res["0"].files:
        if k != "kinds":
            assert np.array_equal(res["0"][k], res["1"][k]), k
