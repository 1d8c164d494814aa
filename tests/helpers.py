"""Shared test helpers (fixtures loading, hashing, conversions)."""
import hashlib
import json
import os

import numpy as np

from oracle import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
CASES = os.path.join(os.path.dirname(HERE), "cases")


def case(name: str) -> str:
    return os.path.join(CASES, name + ".cfg")


def hashes() -> dict:
    with open(os.path.join(GOLDEN, "hashes.json")) as f:
        return json.load(f)


def small() -> dict:
    return dict(np.load(os.path.join(GOLDEN, "small_case.npz")))


def small_mat(d: dict, key: str) -> O.Csr:
    r, c = d[key + "_shape"]
    return O.Csr(int(r), int(c), d[key + "_rp"], d[key + "_ci"], d[key + "_v"])


def small_grid(d: dict) -> dict:
    g = {k: d["grid_" + k] for k in O.RefCase.GRID}
    g["uniform"] = d["grid_uniform"]
    g["h_min"] = float(d["grid_h_min"][0])
    g["nx"], g["ny"] = int(d["dims"][0]), int(d["dims"][1])
    return g


def struct_hash(rows, cols, rp, ci) -> str:
    h = hashlib.sha256()
    h.update(np.asarray([rows, cols], np.int64).tobytes())
    h.update(np.ascontiguousarray(rp, np.int32).tobytes())
    h.update(np.ascontiguousarray(ci, np.int32).tobytes())
    return h.hexdigest()


def value_hash(v) -> str:
    return hashlib.sha256(np.ascontiguousarray(v, np.float64).tobytes()).hexdigest()


def csr_hash(m: O.Csr) -> tuple:
    return struct_hash(m.rows, m.cols, m.rp, m.ci), value_hash(m.v)


def dev_to_csr(M) -> O.Csr:
    """ibm.SparseMatrix -> oracle.Csr (host copy)."""
    rp, ci, v = M.csr()
    return O.Csr(M.rows(), M.cols(), rp, ci, v)


def bench_rhs(spmv, n: int, pin: int = 0):
    """runner.hpp:184-189 consistent right-hand side b = A w."""
    w = np.sin(0.7 * np.arange(n) + 0.3)
    w[pin] = 0.0
    w /= np.sqrt(np.dot(w, w))
    return spmv(w)


def assert_csr_equal(a: O.Csr, b: O.Csr, values: str = "bitwise", rtol: float = 0.0):
    assert (a.rows, a.cols) == (b.rows, b.cols)
    assert np.array_equal(a.rp, b.rp), "row_ptr differs"
    assert np.array_equal(a.ci, b.ci), "col_idx differs"
    if values == "bitwise":
        assert np.array_equal(a.v, b.v), f"values differ (max |d| {np.max(np.abs(a.v - b.v)) if a.nnz else 0})"
    else:
        scale = max(np.max(np.abs(b.v)) if b.nnz else 0.0, 1e-300)
        assert np.max(np.abs(a.v - b.v)) <= rtol * scale if a.nnz else True


def rel_err(a, b):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)) if a.size else 0.0
