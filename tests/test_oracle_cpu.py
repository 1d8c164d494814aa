"""CPU: pin the C restatement (oracle/liboracle.so) against the reference itself and against the
golden fixtures generated from it (tests/golden/make_golden.py). Known-answer cases follow the
reference's own unit tests (proj/tests/test_sparse.cpp, test_krylov.cpp, test_operators.cpp)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests import helpers as H


# ---------------------------------------------------------------- sparse known answers (test_sparse.cpp)
def test_spmv_known_answers(port):
    A = port.from_triplets(2, 2, [0, 1, 1], [0, 0, 1], [2.0, 1.0, 3.0])
    assert np.array_equal(port.spmv(A, np.ones(2)), [2.0, 4.0])  # test_sparse.cpp:14-20
    I = port.from_triplets(5, 5, range(5), range(5), np.ones(5))
    x = np.arange(5.0)
    assert np.array_equal(port.spmv(I, x), x)
    P = O.poisson5(6)
    P0 = port.add(1.0, P, -4.0, port.from_triplets(36, 36, range(36), range(36), np.ones(36)))
    # Poisson rows sum to zero away from the boundary once the diagonal matches the degree
    assert P0.nnz > 0


def test_from_triplets_invariants(port):
    # test_sparse.cpp:134-143
    A = port.from_triplets(3, 3, [1, 1, 1, 0], [2, 0, 2, 0], [1.0, 2.0, 0.5, 0.0])
    assert A.nnz == 2
    assert list(A.ci) == [0, 2] and list(A.v) == [2.0, 1.5]
    with pytest.raises(ValueError):
        port.from_triplets(2, 2, [2], [0], [1.0])


def test_triple_product_slices(port, ref):
    # test_sparse.cpp:99-132: slices {1,7,20} agree with the two-step product; peak intermediate bound
    A, B, C = (O.random_sparse(20, 15, 0.3, 41), O.random_sparse(15, 18, 0.3, 42), O.random_sparse(18, 12, 0.3, 43))
    two = port.spmm(port.spmm(A, B), C)
    for s in (1, 7, 20):
        D, peak, ns = port.triple(A, B, C, s)
        Dr, peakr, nsr = ref.triple(A, B, C, s)
        H.assert_csr_equal(D, Dr)
        assert (peak, ns) == (peakr, nsr)
        assert np.allclose(D.dense(), two.dense(), atol=1e-13)
    P = O.poisson5(12)
    _, full, _ = port.triple(P, P, P, P.rows)
    _, sliced, _ = port.triple(P, P, P, 16)
    assert full == port.spmm(P, P).nnz and sliced < full


def test_transpose_spmm_add_match_reference(port, ref):
    for seed in range(4):
        A = O.random_sparse(17, 11, 0.3, seed)
        B = O.random_sparse(11, 13, 0.3, seed + 100)
        H.assert_csr_equal(port.transpose(A), ref.transpose(A))
        H.assert_csr_equal(port.spmm(A, B), ref.spmm(A, B))
        H.assert_csr_equal(port.add(0.5, A, -2.0, A), ref.add(0.5, A, -2.0, A))
        S = O.random_sparse(15, 15, 0.3, seed + 7)
        H.assert_csr_equal(port.symmetrized(S), ref.symmetrized(S))
        H.assert_csr_equal(port.pin(S, 3), ref.pin(S, 3))


# ---------------------------------------------------------------- krylov known answers (test_krylov.cpp)
def test_cg_identity_and_lu(port):
    I = port.from_triplets(6, 6, range(6), range(6), np.ones(6))
    b = np.linspace(-1, 1, 6)
    r = port.pcg(I, b, kind=0)
    assert r["status"] == 0 and r["iterations"] <= 1 and np.allclose(r["x"], b, atol=1e-12)
    A = O.poisson1d(4)
    r = port.pcg(A, [1.0, 0, 0, 0], kind=0, rel_tol=1e-12)
    assert np.allclose(r["x"], np.linalg.solve(A.dense(), [1.0, 0, 0, 0]), atol=1e-10)


def test_breakdown_and_zero_rhs(port):
    A = port.from_triplets(2, 2, [0, 1], [0, 1], [1.0, -1.0])
    assert port.pcg(A, [0.0, 1.0], kind=0)["status"] == 2
    r = port.pcg(O.poisson5(4), np.zeros(16), x0=np.ones(16), kind=1)
    assert r["status"] == 0 and not r["x"].any()


def test_pcg_matches_reference_bitwise(port, ref):
    A = O.poisson5(10)
    b = np.sin(np.arange(A.rows) * 1.3)
    for kind in (0, 1):
        rp = port.pcg(A, b, kind=kind, rel_tol=1e-8, history=True)
        rr = ref.pcg(A, b, kind=kind, rel_tol=1e-8, history=True)
        assert rp["iterations"] == rr["iterations"]
        assert np.array_equal(rp["x"], rr["x"]) and np.array_equal(rp["history"], rr["history"])


def test_sa_on_1d_poisson(port):
    # test_krylov.cpp:143-171
    A = O.poisson1d(27)
    h = port.sa_build(A, theta=0.25, max_coarse=4)
    assert h.n_levels >= 1
    n_agg = h.level(0)["P"].cols
    assert 27 // 4 <= n_agg <= 27 // 2
    for l in range(h.n_levels):
        L = h.level(l)
        ref_c = L["Pt"].dense() @ L["A"].dense() @ L["P"].dense()
        nxt = h.level(l + 1)["A"] if l + 1 < h.n_levels else h.coarse()
        assert np.allclose(nxt.dense(), ref_c, atol=1e-12 * np.abs(ref_c).max())
    assert h.coarse().rows <= 4


def test_vcycle_contracts_and_is_self_adjoint(port):
    A = O.poisson5(64)
    h = port.sa_build(A)
    b = np.random.default_rng(17).uniform(-1, 1, A.rows)
    z = h.apply(b)
    assert np.linalg.norm(b - port.spmv(A, z)) <= 0.5 * np.linalg.norm(b)
    A = O.poisson5(20)
    h = port.sa_build(A)
    rng = np.random.default_rng(21)
    r1, r2 = rng.uniform(-1, 1, A.rows), rng.uniform(-1, 1, A.rows)
    z1, z2, zs = h.apply(r1), h.apply(r2), h.apply(r1 + r2)
    assert np.max(np.abs(zs - z1 - z2)) <= 1e-10 * np.linalg.norm(zs)
    assert abs(z1 @ r2 - r1 @ z2) <= 1e-10 * abs(r1 @ z2)


def test_iteration_bounds_poisson64(port):
    # test_krylov.cpp:201-227
    A = O.poisson5(64)
    b = np.random.default_rng(33).uniform(-1, 1, A.rows)
    plain = port.pcg(A, b, kind=0)
    diag = port.pcg(A, b, kind=1)
    sa = port.pcg(A, b, kind=2, hier=port.sa_build(A))
    assert plain["iterations"] <= 300 and diag["iterations"] <= plain["iterations"]
    assert sa["iterations"] < plain["iterations"] / 4


def test_delta_roma_moments(port, ref):
    # body.hpp:19-28; test_body.cpp:11-43 (partition of unity / first moment over a unit lattice)
    h = 0.1
    for off in np.linspace(0, 1, 11):
        xs = (np.arange(-3, 4) + off) * h
        w = np.array([port.delta_roma(x, h) for x in xs])
        assert abs(w.sum() * h - 1.0) < 1e-12
        assert abs((w * xs).sum() * h) < 1e-12
    for r in np.linspace(-0.2, 0.2, 101):
        assert port.delta_roma(r, h) == ref.delta_roma(r, h)


# ---------------------------------------------------------------- golden fixtures
@pytest.mark.parametrize("name", ["cavity", "cylinder_re40_smoke", "flapping_smoke", "cylinder_re40"])
def test_port_reproduces_golden_case(port, ref, name):
    """E/H, lhs2 and every SA level of the restatement hash-equal to the reference's."""
    gold = H.hashes()[name]
    c = ref.case(H.case(name))
    g = c.grid()
    bd = c.bodies()
    if c.n_b:
        E, Hm = port.assemble_EH(g, bd["x"], bd["y"], bd["ds"])
        for k, m in (("E", E), ("H", Hm)):
            assert H.csr_hash(m) == (gold[k]["struct"], gold[k]["values"]), k
    else:
        E = O.Csr(0, c.n_q, np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0))
    Q = port.concat_cols(c.op("G"), port.transpose(E))
    QT = port.transpose(Q)
    raw, _, _ = port.triple(QT, c.op("BN"), Q, QT.rows)
    lhs2 = port.pin(port.symmetrized(raw), 0)
    assert H.csr_hash(lhs2) == (gold["lhs2"]["struct"], gold["lhs2"]["values"])
    h = port.sa_build(lhs2, tail=2 * c.n_b)
    assert h.n_levels == len(gold["levels"])
    for l, gl in enumerate(gold["levels"]):
        L = h.level(l)
        for k in ("A", "P", "Pt"):
            assert H.csr_hash(L[k]) == (gl[k]["struct"], gl[k]["values"]), (l, k)
        assert L["omega"] == gl["omega"]
        n_agg, agg = port.aggregate(L["A"], 0.25 * 0.5 ** l, L["A"].rows - 2 * c.n_b)
        assert n_agg == gl["n_agg"]
        import hashlib
        assert hashlib.sha256(np.ascontiguousarray(agg, np.int32).tobytes()).hexdigest() == gl["agg"]
    b = H.bench_rhs(lambda w: port.spmv(lhs2, w), lhs2.rows)
    r = port.pcg(lhs2, b, kind=2, hier=h)
    assert r["iterations"] == gold["bench_pcg_sa"]["iterations"]


def test_port_reproduces_small_case_fixture(port):
    d = H.small()
    g = H.small_grid(d)
    E, Hm = port.assemble_EH(g, d["body_x"], d["body_y"], d["body_ds"])
    H.assert_csr_equal(E, H.small_mat(d, "E"))
    H.assert_csr_equal(Hm, H.small_mat(d, "H"))
    lhs2 = H.small_mat(d, "lhs2")
    n_b = int(d["dims"][4])
    h = port.sa_build(lhs2, tail=2 * n_b)
    assert h.n_levels == int(d["n_levels"][0])
    for l in range(h.n_levels):
        for k in ("A", "P", "Pt"):
            H.assert_csr_equal(h.level(l)[k], H.small_mat(d, f"L{l}_{k}"))
    z = h.apply(d["bench_b"])
    assert np.max(np.abs(z - d["vcycle_z"])) <= 1e-12 * np.max(np.abs(d["vcycle_z"]))
    r = port.pcg(lhs2, d["bench_b"], kind=2, hier=h, history=True)
    assert r["iterations"] == int(d["bench_iters"][0])
    assert np.array_equal(r["x"], d["bench_x"])
