"""GPU parity: structural sparse kernels vs the C restatement (bit-exact structure AND values —
the device reproduces the reference's accumulation order without FMA contraction)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1109_3524_b200 import ibm
from tests import helpers as H

pytestmark = pytest.mark.gpu


def dev(m):
    return ibm.SparseMatrix.from_host(m)


def mats():
    d = H.small()
    return [O.poisson5(33), O.random_sparse(57, 41, 0.15, 1), H.small_mat(d, "lhs2"), H.small_mat(d, "E"),
            H.small_mat(d, "QT"), H.small_mat(d, "L1_A")]


def test_spmv_bitwise(port):
    """Short-row matrices (SELL-32, thread per row, column-order non-FMA sums) are bit-exact with
    spmv_into; long-row Galerkin levels use the CSR-vector kernel (lane-strided sums): 1e-14."""
    for m in mats():
        x = np.sin(np.arange(m.cols) * 0.37 + 0.1)
        y = dev(m).spmv(x)
        yo = port.spmv(m, x)
        if m.nnz <= 12 * m.rows:
            assert np.array_equal(y, yo)
        else:
            assert np.max(np.abs(y - yo)) <= 1e-14 * np.max(np.abs(m.v)) * np.sum(np.abs(x))


@pytest.mark.parametrize("n_long", [1, 7, 40])
def test_spmv_hybrid_long_rows_bitwise(port, n_long):
    """SELL-32-sigma with a few rows of > 96 entries (the Galerkin body tail): the long rows run
    one warp each with an in-order sum, so the whole product stays bit-exact with spmv_into."""
    rng = np.random.default_rng(11 + n_long)
    n = 4000  # mean row length <= 8 keeps the thread-per-row plan at this size
    rows, cols, vals = [], [], []
    long_ids = set(rng.choice(n, n_long, replace=False).tolist())
    for i in range(n):
        k = int(rng.integers(97, 130)) if i in long_ids else int(rng.integers(1, 12))
        c = np.sort(rng.choice(n, size=k, replace=False))
        rows += [i] * k
        cols += c.tolist()
        vals += rng.uniform(-1, 1, k).tolist()
    m = port.from_triplets(n, n, np.array(rows), np.array(cols), np.array(vals))
    x = rng.uniform(-1, 1, n)
    for xv in (x, np.sin(np.arange(n) * 0.37 + 0.1)):
        assert np.array_equal(dev(m).spmv(xv), port.spmv(m, xv))


def test_spmv_known_answers():
    A = ibm.SparseMatrix.from_triplets(2, 2, [(0, 0, 2.0), (1, 0, 1.0), (1, 1, 3.0)])
    assert np.array_equal(A.spmv(np.ones(2)), [2.0, 4.0])
    with pytest.raises(ValueError):
        A.spmv(np.ones(3))


def test_from_triplets_invariants():
    A = ibm.SparseMatrix.from_triplets(3, 3, [(1, 2, 1.0), (1, 0, 2.0), (1, 2, 0.5), (0, 0, 0.0)])
    rp, ci, v = A.csr()
    assert A.nnz() == 2 and list(ci) == [0, 2] and list(v) == [2.0, 1.5]
    with pytest.raises(ValueError):
        ibm.SparseMatrix.from_triplets(2, 2, [(2, 0, 1.0)])


def test_transpose_bitwise(port):
    for m in mats():
        H.assert_csr_equal(H.dev_to_csr(dev(m).transpose()), port.transpose(m))


def test_spmm_bitwise(port):
    for seed in range(3):
        A = O.random_sparse(40, 30, 0.2, seed)
        B = O.random_sparse(30, 35, 0.2, seed + 50)
        H.assert_csr_equal(H.dev_to_csr(ibm.spmm(dev(A), dev(B))), port.spmm(A, B))
    P = O.poisson5(20)
    H.assert_csr_equal(H.dev_to_csr(ibm.spmm(dev(P), dev(P))), port.spmm(P, P))
    with pytest.raises(ValueError):
        ibm.spmm(dev(O.random_sparse(3, 4, 0.5, 1)), dev(O.random_sparse(3, 4, 0.5, 2)))


@pytest.mark.parametrize("slice_rows", [1, 7, 20, 1000])
def test_triple_product_bitwise(port, slice_rows):
    A, B, Cm = (O.random_sparse(20, 15, 0.3, 41), O.random_sparse(15, 18, 0.3, 42), O.random_sparse(18, 12, 0.3, 43))
    st = ibm.TripleProductStats()
    D = ibm.sliced_triple_product(dev(A), dev(B), dev(Cm), slice_rows, st)
    Do, peak, ns = port.triple(A, B, Cm, slice_rows)
    H.assert_csr_equal(H.dev_to_csr(D), Do)
    assert (st.peak_slice_nnz, st.slices) == (peak, ns)


def test_galerkin_triple_bitwise(port):
    d = H.small()
    Pt, A, P = H.small_mat(d, "L0_Pt"), H.small_mat(d, "L0_A"), H.small_mat(d, "L0_P")
    D = ibm.sliced_triple_product(dev(Pt), dev(A), dev(P), Pt.rows)
    H.assert_csr_equal(H.dev_to_csr(D), H.small_mat(d, "L1_A"))


def test_add_symmetrize_pin_bitwise(port):
    for seed in range(3):
        S = O.random_sparse(30, 30, 0.2, seed + 9)
        T = O.random_sparse(30, 30, 0.2, seed + 19)
        H.assert_csr_equal(H.dev_to_csr(ibm.add_sparse(0.5, dev(S), -1.25, dev(T))), port.add(0.5, S, -1.25, T))
        H.assert_csr_equal(H.dev_to_csr(ibm.add_sparse(1.0, dev(S), -1.0, dev(S))), port.add(1.0, S, -1.0, S))
        H.assert_csr_equal(H.dev_to_csr(ibm.symmetrized(dev(S))), port.symmetrized(S))
        H.assert_csr_equal(H.dev_to_csr(ibm.pin_row_col(dev(S), 4)), port.pin(S, 4))
    L2 = H.small_mat(H.small(), "lhs2")
    assert ibm.is_symmetric(dev(L2), 1e-12)
    assert not ibm.is_symmetric(dev(O.random_sparse(10, 10, 0.4, 3)), 1e-12)


def test_scaled_variants(port):
    m = O.random_sparse(25, 19, 0.3, 5)
    d_r = np.linspace(0.5, 2.0, 25)
    d_c = np.linspace(-1.0, 3.0, 19)
    A = dev(m)
    H.assert_csr_equal(H.dev_to_csr(A.scaled(0.3)), O.Csr(m.rows, m.cols, m.rp, m.ci, m.v * 0.3))
    rows = np.repeat(np.arange(m.rows), np.diff(m.rp))
    H.assert_csr_equal(H.dev_to_csr(A.scaled_rows(d_r)), O.Csr(m.rows, m.cols, m.rp, m.ci, m.v * d_r[rows]))
    H.assert_csr_equal(H.dev_to_csr(A.scaled_cols(d_c)), O.Csr(m.rows, m.cols, m.rp, m.ci, m.v * d_c[m.ci]))


def test_empty_and_ragged():
    Z = ibm.SparseMatrix.from_triplets(4, 3, [])
    assert Z.nnz() == 0
    assert np.array_equal(Z.spmv(np.ones(3)), np.zeros(4))
    T = Z.transpose()
    assert (T.rows(), T.cols(), T.nnz()) == (3, 4, 0)
    R = ibm.SparseMatrix.from_triplets(5, 5, [(0, 4, 1.0), (4, 0, 2.0)])
    assert np.array_equal(R.spmv(np.arange(5.0)), [4.0, 0, 0, 0, 0])


@pytest.mark.parametrize("op", ["lhs2", "A", "L", "QT"])
def test_stencil_format_spmv_bitwise(port, ref, op):
    """Stencil (DIA-hybrid) plan on the 330^2 case operators: lhs2 (one stride + body extras and
    generic body rows), A and L (two strides: u rows nx-1, v rows nx). Bit-exact vs spmv_into."""
    c = ref.case(H.case("cylinder_re40"))
    m = c.op(op)
    x = np.cos(np.arange(m.cols) * 0.61 + 0.2)
    assert np.array_equal(dev(m).spmv(x), port.spmv(m, x))


def test_spmm_hash_and_long_row_paths_bitwise(port):
    """Both SpGEMM paths against spmm_rows (sparse.hpp:226-268): rows averaging >= 32 products go
    through the warp hash accumulator, and a row of more than 131k products through ESC (placed
    back into the hash result). Gustavson-order sums, cancelled entries kept: bit-exact."""
    rng = np.random.default_rng(17)
    m, k, n = 60, 400, 500
    ra, ca, va = [], [], []
    for i in range(m):
        cols = np.arange(k) if i == 7 else np.sort(rng.choice(k, 40, replace=False))
        ra += [i] * len(cols)
        ca += cols.tolist()
        va += rng.uniform(-1, 1, len(cols)).tolist()
    rb, cb, vb = [], [], []
    for i in range(k):
        cols = np.sort(rng.choice(n, 420, replace=False))
        rb += [i] * len(cols)
        cb += cols.tolist()
        vb += rng.choice([-1.0, 1.0, 0.5, -0.5], len(cols)).tolist()  # exact cancellations occur
    A = port.from_triplets(m, k, np.array(ra), np.array(ca), np.array(va))
    B = port.from_triplets(k, n, np.array(rb), np.array(cb), np.array(vb))
    C = ibm.spmm(dev(A), dev(B))
    H.assert_csr_equal(H.dev_to_csr(C), port.spmm(A, B))
