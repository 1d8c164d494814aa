"""Race detection by repetition (compute-sanitizer is closed on this GPU pool: its runs left GPUs
needing a reset). Every reduction on the path is deterministic by design — block partials summed in
fixed order by a finalize kernel, self-resetting arrival counters, warp-ordered hash SpGEMM
accumulation, the exact parallel greedy aggregation — so a data race or a stale-counter bug shows
up as a run-to-run difference. Each object is rebuilt / re-solved several times, with other work
interleaved so scheduling differs, and must come out bit-identical."""
import hashlib

import numpy as np
import pytest

from paper_1109_3524_b200 import ibm
from tests import helpers as H

pytestmark = pytest.mark.gpu


def _hier_digest(h):
    d = hashlib.sha256()
    for l in range(h.n_levels):
        lv = h.level(l)
        for k in ("A", "P", "Pt"):
            rp, ci, v = lv[k].csr()
            for a in (rp, ci, v):
                d.update(np.ascontiguousarray(a).tobytes())
        d.update(np.float64(lv["omega"]).tobytes())
        n, agg = h.aggregates(l)
        d.update(np.ascontiguousarray(agg[: lv["A"].rows()], np.int32).tobytes())
    rp, ci, v = h.coarse_A().csr()
    for a in (rp, ci, v):
        d.update(np.ascontiguousarray(a).tobytes())
    return d.hexdigest()


@pytest.mark.parametrize("name,h_min", [("flapping", 0.0), ("cylinder_re40", 0.002)])
def test_hierarchy_build_and_solve_repeat_bitwise(name, h_min):
    st = ibm.Stepper(H.case(name), h_min=h_min)
    A = st.op("lhs2")
    b = H.bench_rhs(A.spmv, A.rows())
    digests, xs, its = [], [], []
    for k in range(4):
        h = ibm.build_sa_hierarchy(A, ibm.SaOptions(keep_fine_tail=2 * st.n_b))
        digests.append(_hier_digest(h))
        r = ibm.pcg(A, b, None, ibm.SaPreconditioner(h), ibm.SolverParams())
        xs.append(r.x)
        its.append(r.iterations)
        # interleave unrelated device work so the next build is scheduled differently
        ibm.spmm(A, A)
    assert len(set(digests)) == 1, digests
    assert len(set(its)) == 1, its
    assert all(np.array_equal(xs[0], x) for x in xs[1:])


def test_moving_body_steps_repeat_bitwise():
    """Refresh (incremental lhs2), SA rebuild with cached aggregates, both graph solves: two
    independent steppers produce bit-identical trajectories."""
    runs = []
    for _ in range(2):
        st = ibm.Stepper(H.case("flapping_smoke"))
        out = []
        for _ in range(6):
            r = st.advance()
            assert r.ok, r.message
            out.append((r.solve1_iters, r.solve2_iters, st.get("q").tobytes(), st.get("lambda").tobytes()))
        runs.append(out)
    assert runs[0] == runs[1]
