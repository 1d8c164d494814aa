"""GPU parity: delta_roma, E/H assembly and the coupled system — bit-exact sparsity and values
(SURVEY §7 hard part 2: FMA contraction would change the E / lhs2 structure)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1109_3524_b200 import ibm
from tests import helpers as H

pytestmark = pytest.mark.gpu


def test_delta_roma_bitwise(port):
    h = 0.02
    r = np.concatenate([np.linspace(-0.04, 0.04, 4001), [0.5 * h, -0.5 * h, 1.5 * h, -1.5 * h, 1.5 * h * (1 - 1e-16)]])
    d = ibm.delta_roma(r, h)
    assert np.array_equal(d, [port.delta_roma(x, h) for x in r])


def test_EH_small_case_bitwise():
    d = H.small()
    E, Hm = ibm.assemble_interpolation_regularization(H.small_grid(d), d["body_x"], d["body_y"], d["body_ds"])
    H.assert_csr_equal(H.dev_to_csr(E), H.small_mat(d, "E"))
    H.assert_csr_equal(H.dev_to_csr(Hm), H.small_mat(d, "H"))


@pytest.mark.parametrize("name", ["cylinder_re40_smoke", "flapping_smoke", "cylinder_re40"])
def test_EH_and_lhs2_match_golden(ref, name):
    gold = H.hashes()[name]
    c = ref.case(H.case(name))
    g = c.grid()
    bd = c.bodies()
    E, Hm = ibm.assemble_interpolation_regularization(g, bd["x"], bd["y"], bd["ds"])
    assert H.csr_hash(H.dev_to_csr(E)) == (gold["E"]["struct"], gold["E"]["values"])
    assert H.csr_hash(H.dev_to_csr(Hm)) == (gold["H"]["struct"], gold["H"]["values"])
    G = ibm.SparseMatrix.from_host(c.op("G"))
    BN = ibm.SparseMatrix.from_host(c.op("BN"))
    Q, QT, L2 = ibm.assemble_coupled_system(G, E, BN, 0, 0)
    for k, m in (("Q", Q), ("QT", QT), ("lhs2", L2)):
        assert H.csr_hash(H.dev_to_csr(m)) == (gold[k]["struct"], gold[k]["values"]), k


def test_coupled_system_sliced_equals_full(ref):
    c = ref.case(H.case("flapping_smoke"))
    g = c.grid()
    bd = c.bodies()
    E, _ = ibm.assemble_interpolation_regularization(g, bd["x"], bd["y"], bd["ds"])
    G = ibm.SparseMatrix.from_host(c.op("G"))
    BN = ibm.SparseMatrix.from_host(c.op("BN"))
    full = H.dev_to_csr(ibm.assemble_coupled_system(G, E, BN, 0, 0)[2])
    st = ibm.TripleProductStats()
    sliced = H.dev_to_csr(ibm.assemble_coupled_system(G, E, BN, 0, 1000, st)[2])
    H.assert_csr_equal(sliced, full)
    assert 0 < st.peak_slice_nnz


def test_support_outside_uniform_region_rejected():
    d = H.small()
    g = H.small_grid(d)
    x = np.array([g["uniform"][1] - 0.1 * g["h_min"]])
    with pytest.raises(RuntimeError, match="uniform"):
        ibm.assemble_interpolation_regularization(g, x, np.zeros(1), np.ones(1))


def test_interpolation_reproduces_linear_fields():
    # test_operators.cpp:139-205: partition of unity, constant and linear reproduction
    d = H.small()
    g = H.small_grid(d)
    nx, ny = g["nx"], g["ny"]
    xs = np.array([0.013, -0.37])
    ys = np.array([0.21, 0.05])
    E, _ = ibm.assemble_interpolation_regularization(g, xs, ys, np.full(2, 0.1))
    fu = lambda x, y: 0.7 * x - 1.3 * y + 0.2
    fv = lambda x, y: 1.1 * x + 0.4 * y - 1.0
    q = np.zeros(E.cols())
    n_u = (nx - 1) * ny
    for j in range(ny):
        for i_f in range(1, nx):
            q[(i_f - 1) + j * (nx - 1)] = fu(g["x_faces"][i_f], g["y_c"][j]) * g["dy"][j]
    for j_f in range(1, ny):
        for i in range(nx):
            q[n_u + i + (j_f - 1) * nx] = fv(g["x_c"][i], g["y_faces"][j_f]) * g["dx"][i]
    eq = E.spmv(q)
    assert np.allclose(eq[:2], fu(xs, ys), atol=1e-10)
    assert np.allclose(eq[2:], fv(xs, ys), atol=1e-10)
