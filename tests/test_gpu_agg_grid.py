"""Pass 1 of the greedy aggregation on grid-shaped strength graphs (amg_setup.cu k_greedy_grid):
lines pipelined two columns apart, 32 per warp. It must give exactly the reference's aggregates
(sa_detail::aggregate, amg.hpp:79-107) — on the golden level-0 operators and on random 5-point
grids with directed (non-symmetric) strength, dropped edges, and sizes that are not multiples of
the warp / window widths."""
import ctypes as C
import hashlib

import numpy as np
import pytest

from oracle import oracle as O
from paper_1109_3524_b200 import ibm
from tests import helpers as H

pytestmark = pytest.mark.gpu


def _agg(Ad, theta, n_core):
    agg = np.zeros(max(n_core, 1), np.int32)
    n = C.c_int()
    Ad.ctx.check(Ad.ctx.lib.ibmgpu_aggregate(Ad.ctx.h, Ad.h, theta, n_core, agg.ctypes.data_as(C.POINTER(C.c_int)),
                                             C.byref(n)))
    return n.value, agg[:n_core]


def _planned(m):
    Ad = ibm.SparseMatrix.from_host(m)
    Ad.spmv(np.zeros(m.cols))  # builds the SpMV plan (stencil: the stride the grid pass-1 uses)
    return Ad


@pytest.mark.parametrize("name", ["cylinder_re40_smoke", "flapping_smoke", "cylinder_re40"])
def test_grid_pass1_matches_golden_level0(ref, name, monkeypatch):
    gold = H.hashes()[name]["levels"][0]
    c = ref.case(H.case(name))
    A = c.hierarchy().level(0)["A"]
    n_core = A.rows - 2 * c.n_b
    Ad = _planned(A)
    assert Ad.format_bytes()[1] == 3  # stencil plan
    for kernel in ("grid", "lfmis"):
        monkeypatch.setenv("IBMGPU_AGG", kernel)
        n, agg = _agg(Ad, 0.25, n_core)
        assert n == gold["n_agg"], kernel
        assert hashlib.sha256(np.ascontiguousarray(agg, np.int32).tobytes()).hexdigest() == gold["agg"], kernel


def _csr(n, r, c, v):
    order = np.lexsort((c, r))
    r, c, v = np.asarray(r)[order], np.asarray(c, np.int32)[order], np.asarray(v, np.float64)[order]
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    return O.Csr(n, n, np.cumsum(rp).astype(np.int32), c, v)


def _grid5(S, NY, seed, drop):
    """5-point pattern, random magnitudes (non-symmetric), some couplings weakened below theta."""
    rng = np.random.default_rng(seed)
    n = S * NY
    rows, cols, vals = [], [], []
    for off, ok in ((-S, lambda i: i >= S), (-1, lambda i: i % S > 0), (1, lambda i: i % S < S - 1),
                    (S, lambda i: i + S < n)):
        i = np.arange(n)
        i = i[ok(i)]
        v = -rng.uniform(0.5, 1.5, len(i))
        weak = rng.random(len(i)) < drop
        v[weak] *= 1e-3
        rows.append(i), cols.append(i + off), vals.append(v)
    rows.append(np.arange(n)), cols.append(np.arange(n)), vals.append(rng.uniform(3.5, 4.5, n))
    r, cc, v = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
    return _csr(n, r, cc, v)


@pytest.mark.parametrize("S,NY,seed,drop", [(4097, 40, 1, 0.0), (1000, 70, 2, 0.2), (333, 129, 3, 0.5),
                                            (2, 4096, 4, 0.3), (5000, 33, 5, 0.05), (64, 2048, 6, 0.7)])
def test_grid_pass1_random_grids(port, monkeypatch, S, NY, seed, drop):
    A = _grid5(S, NY, seed, drop)
    n = S * NY
    n_ref, agg_ref = port.aggregate(A, 0.25, n)
    Ad = _planned(A)
    for kernel in ("grid", "lfmis"):
        monkeypatch.setenv("IBMGPU_AGG", kernel)
        n_dev, agg_dev = _agg(Ad, 0.25, n)
        assert n_dev == n_ref, (kernel, n_dev, n_ref)
        assert np.array_equal(agg_dev, np.asarray(agg_ref, np.int32)[:n]), kernel


def test_grid_pass1_falls_back_on_a_wrapping_edge(port, monkeypatch):
    """A strength edge that wraps across a grid line is not grid-shaped: the general kernel runs and
    the result is still the reference's."""
    A = _grid5(300, 20, 9, 0.1)
    r = np.repeat(np.arange(A.rows), np.diff(A.rp))
    i = 4 * 300 - 1  # end of line 3 <-> start of line 4, strongly coupled across the line break
    B = _csr(A.rows, np.concatenate([r, [i, i + 1]]), np.concatenate([A.ci, [i + 1, i]]),
             np.concatenate([A.v, [-1.0, -1.0]]))
    n_ref, agg_ref = port.aggregate(B, 0.25, B.rows)
    monkeypatch.setenv("IBMGPU_AGG", "grid")
    n_dev, agg_dev = _agg(_planned(B), 0.25, B.rows)
    assert n_dev == n_ref and np.array_equal(agg_dev, np.asarray(agg_ref, np.int32)[:B.rows])
