"""GPU parity of the row-slab distributed PCG (csrc/dist.cu). The partition is
emulated on the one GPU (loopback communicator: every rank's kernels run on this device, halos move
by device copies; no kernel waits on another rank's). Contract: iterations within ±2 of the
single-GPU solve and of the reference, solutions within 1e-6 relative at the reference tolerance,
and the initial residual (one distributed SpMV + an allreduced norm) equal to the single-GPU one
to rounding."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1109_3524_b200 import ibm
from tests import helpers as H

pytestmark = pytest.mark.gpu


def _cell_j(y_faces, y):
    return np.clip(np.searchsorted(y_faces, y, side="right") - 1, 0, len(y_faces) - 2).astype(np.int32)


@pytest.fixture(scope="module")
def small():
    d = H.small()
    n_b = int(d["dims"][4])
    A = ibm.SparseMatrix.from_host(H.small_mat(d, "lhs2"))
    h = ibm.build_sa_hierarchy(A, ibm.SaOptions(keep_fine_tail=2 * n_b))
    single = ibm.pcg(A, d["bench_b"], None, ibm.SaPreconditioner(h), ibm.SolverParams(record_history=True))
    return d, A, h, single


@pytest.mark.parametrize("R,min_rows", [(1, 0), (2, 0), (3, 0), (4, 0), (2, 1000), (4, 10 ** 9)])
def test_loopback_sa_small_case(small, R, min_rows):
    d, A, h, single = small
    nx, ny = int(d["dims"][0]), int(d["dims"][1])
    owner = ibm.partition_lambda(nx, ny, _cell_j(d["grid_y_faces"], d["body_y"]), R)
    ds = ibm.DistSolver(A, ibm.SaPreconditioner(h), owner, virtual_ranks=R, min_dist_rows=min_rows)
    info = ds.info()
    assert info["nranks"] == R and info["local_ranks"] == R and info["loopback"] == 1
    assert info["dist_levels"] >= 1
    if R > 1:
        assert info["halo"] > 0
    r = ds.solve(d["bench_b"], params=ibm.SolverParams(record_history=True))
    assert r.converged()
    assert abs(r.iterations - single.iterations) <= 2
    assert abs(r.iterations - int(d["bench_iters"][0])) <= 2
    assert abs(r.history[0] - single.history[0]) <= 1e-13 * single.history[0]
    assert np.max(np.abs(r.x - d["bench_x"])) <= 1e-6 * np.max(np.abs(d["bench_x"]))
    # repeated solves reuse the plans
    r2 = ds.solve(d["bench_b"])
    assert r2.iterations == r.iterations and np.array_equal(r2.x, r.x)


@pytest.mark.parametrize("kind", ["identity", "diagonal"])
def test_loopback_diag_identity_poisson(kind):
    A = O.poisson5(40)
    Ad = ibm.SparseMatrix.from_host(A)
    b = np.random.default_rng(5).uniform(-1, 1, A.rows)
    M = ibm.IdentityPreconditioner() if kind == "identity" else ibm.DiagonalPreconditioner(Ad)
    single = ibm.pcg(Ad, b, None, M, ibm.SolverParams())
    for R in (2, 3):
        r = ibm.DistSolver(Ad, M, ibm.block_partition(A.rows, R), virtual_ranks=R).solve(b)
        assert r.converged() and abs(r.iterations - single.iterations) <= 2
        assert np.max(np.abs(r.x - single.x)) <= 1e-6 * np.max(np.abs(single.x))


def test_loopback_ranks_without_rows(small):
    d, A, h, single = small
    owner = np.zeros(A.rows(), np.int32)
    owner[-5:] = 2  # rank 1 owns nothing, rank 2 a few force rows
    r = ibm.DistSolver(A, ibm.SaPreconditioner(h), owner, virtual_ranks=3).solve(d["bench_b"])
    assert r.converged() and abs(r.iterations - single.iterations) <= 2
    assert np.max(np.abs(r.x - d["bench_x"])) <= 1e-6 * np.max(np.abs(d["bench_x"]))


def test_loopback_nonzero_x0_and_zero_rhs(small):
    d, A, h, single = small
    owner = ibm.block_partition(A.rows(), 2)
    ds = ibm.DistSolver(A, ibm.SaPreconditioner(h), owner, virtual_ranks=2)
    r0 = ds.solve(np.zeros(A.rows()), x0=np.ones(A.rows()))
    assert r0.converged() and r0.iterations == 0 and not np.any(r0.x)  # krylov.hpp:85-89
    x0 = 0.5 * d["bench_x"]
    r = ds.solve(d["bench_b"], x0=x0)
    rs = ibm.pcg(A, d["bench_b"], x0, ibm.SaPreconditioner(h), ibm.SolverParams())
    assert abs(r.iterations - rs.iterations) <= 2


def test_dist_argument_errors(small):
    d, A, h, single = small
    with pytest.raises(ValueError):
        ibm.DistSolver(A, ibm.SaPreconditioner(h), np.full(A.rows(), 5, np.int32), virtual_ranks=2)
    with pytest.raises(ValueError):
        ibm.DistSolver(A, ibm.SaPreconditioner(h), np.zeros(3, np.int32), virtual_ranks=2)
    B = ibm.SparseMatrix.from_host(O.poisson5(4))
    h1 = ibm.build_sa_hierarchy(B)  # 16 rows <= max_coarse: no levels
    with pytest.raises(RuntimeError, match="no levels"):
        ibm.DistSolver(B, ibm.SaPreconditioner(h1), np.zeros(16, np.int32), virtual_ranks=2)


def test_loopback_full_size_c2():
    """C2 (1042^2 + cylinder): 4 emulated slabs, fine levels distributed, tail replicated."""
    import json
    import os
    with open(os.path.join(H.GOLDEN, "hashes_large.json")) as f:
        g = json.load(f)["c2"]
    st = ibm.Stepper(H.case("cylinder_re40"), h_min=0.002, dt=0.001)
    A = st.op("lhs2")
    b = H.bench_rhs(A.spmv, A.rows())
    owner = ibm.partition_lambda(st.nx, st.ny, _cell_j(st.grid()["y_faces"], st.bodies()["y"]), 4)
    ds = ibm.DistSolver(A, ibm.SaPreconditioner(st.hierarchy()), owner, virtual_ranks=4, min_dist_rows=100000)
    assert ds.info()["dist_levels"] >= 2
    r = ds.solve(b)
    assert r.converged() and abs(r.iterations - g["bench_pcg_sa"]["iterations"]) <= 2
    rs = ibm.pcg(A, b, None, ibm.SaPreconditioner(st.hierarchy()), ibm.SolverParams())
    assert np.linalg.norm(r.x - rs.x) <= 1e-5 * np.linalg.norm(rs.x)


@pytest.mark.parametrize("name,steps", [("cylinder_re40_smoke", 3), ("flapping_smoke", 3), ("cavity", 2)])
def test_distributed_stepper_matches_single(name, steps):
    """Stepper with both solves row-slab distributed over 3 emulated ranks vs the single-GPU stepper
    (moving bodies re-plan solve 2 every step)."""
    a = ibm.Stepper(H.case(name))
    b = ibm.Stepper(H.case(name))
    b.distribute(virtual_ranks=3, min_dist_rows=0)
    for _ in range(steps):
        ra, rb = a.advance(), b.advance()
        assert ra.ok and rb.ok, (ra.message, rb.message)
        assert abs(ra.solve2_iters - rb.solve2_iters) <= 2 and abs(ra.solve1_iters - rb.solve1_iters) <= 2
    qa, qb = a.get("q"), b.get("q")
    la, lb = a.get("lambda"), b.get("lambda")
    assert np.linalg.norm(qa - qb) <= 1e-6 * np.linalg.norm(qa)
    assert np.linalg.norm(la - lb) <= 1e-6 * max(np.linalg.norm(la), 1e-300)
    if a.n_b:
        fa, fb = a.forces(), b.forces()
        assert abs(fa["cd"] - fb["cd"]) <= 1e-6 * abs(fa["cd"])
    b.distribute(0)  # back to the single-GPU graph solve
    assert b.advance().ok


def test_nccl_backend_one_rank(small):
    """The NCCL code path on the one GPU available: a one-rank communicator, so every allreduce
    and the final gather of x go through ncclAllReduce (captured in the per-iteration graph)."""
    d, A, h, single = small
    ctx = ibm.Context(0, nranks=1, rank=0, nccl_id=ibm.nccl_unique_id())
    A1 = ibm.SparseMatrix.from_host(H.small_mat(d, "lhs2"), ctx=ctx)
    n_b = int(d["dims"][4])
    h1 = ibm.build_sa_hierarchy(A1, ibm.SaOptions(keep_fine_tail=2 * n_b))
    ds = ibm.DistSolver(A1, ibm.SaPreconditioner(h1), np.zeros(A1.rows(), np.int32))
    assert ds.info()["loopback"] == 0 and ds.info()["nranks"] == 1
    r = ds.solve(d["bench_b"])
    assert r.converged() and abs(r.iterations - single.iterations) <= 2
    assert np.max(np.abs(r.x - d["bench_x"])) <= 1e-6 * np.max(np.abs(d["bench_x"]))
    st = ibm.Stepper(H.case("cylinder_re40_smoke"), ctx=ctx)
    ref = ibm.Stepper(H.case("cylinder_re40_smoke"))
    st.distribute(virtual_ranks=1, min_dist_rows=0)
    for _ in range(2):
        ra, rb = ref.advance(), st.advance()
        assert ra.ok and rb.ok and abs(ra.solve2_iters - rb.solve2_iters) <= 2
    la, lb = ref.get("lambda"), st.get("lambda")
    assert np.linalg.norm(la - lb) <= 1e-6 * np.linalg.norm(la)


@pytest.mark.parametrize("R", [2, 4])
def test_nccl_p2p_halos_match_device_copies(small, R):
    """The ncclSend/ncclRecv halo path on one GPU: a one-rank communicator with R virtual ranks
    moves every halo as NCCL send/recv pairs to self (captured in the per-iteration graph). The
    result must be bitwise the device-copy loopback's, for the coupled SA solve and for two
    distributed Stepper steps (both solves)."""
    d, A, h, single = small
    nx, ny = int(d["dims"][0]), int(d["dims"][1])
    owner = ibm.partition_lambda(nx, ny, _cell_j(d["grid_y_faces"], d["body_y"]), R)
    ref = ibm.DistSolver(A, ibm.SaPreconditioner(h), owner, virtual_ranks=R).solve(d["bench_b"])
    ctx = ibm.Context(0, nranks=1, rank=0, nccl_id=ibm.nccl_unique_id())
    A1 = ibm.SparseMatrix.from_host(H.small_mat(d, "lhs2"), ctx=ctx)
    h1 = ibm.build_sa_hierarchy(A1, ibm.SaOptions(keep_fine_tail=2 * int(d["dims"][4])))
    ds = ibm.DistSolver(A1, ibm.SaPreconditioner(h1), owner, virtual_ranks=R)
    info = ds.info()
    assert info["loopback"] == 2 and info["nranks"] == R and info["halo"] > 0
    r = ds.solve(d["bench_b"])
    assert r.iterations == ref.iterations and np.array_equal(r.x, ref.x)
    sa, sb = ibm.Stepper(H.case("cylinder_re40_smoke")), ibm.Stepper(H.case("cylinder_re40_smoke"), ctx=ctx)
    sa.distribute(virtual_ranks=R, min_dist_rows=0)
    sb.distribute(virtual_ranks=R, min_dist_rows=0)
    for _ in range(2):
        ra, rb = sa.advance(), sb.advance()
        assert ra.ok and rb.ok and ra.solve2_iters == rb.solve2_iters
    for f in ("q", "lambda"):
        assert np.array_equal(sa.get(f), sb.get(f))
