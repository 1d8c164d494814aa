"""Generate the golden fixtures from the unmodified reference (oracle/_ref/libibmref.so).

Run in the build container (where /root/reference exists):  python tests/golden/make_golden.py
Outputs (committed):
  tests/golden/small_case.npz  full operators / hierarchy / 3 steps of a 64^2 uniform cylinder
  tests/golden/hashes.json     sha256 of CSR structures, value checksums, SA level data and
                               first-step results for the bundled cases
The reference itself publishes no golden data; these vectors are produced by
running its own code paths (parse_config -> Stepper ctor -> advance, build_sa_hierarchy,
sa_detail::aggregate, pcg) on deterministic inputs.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

CASES = os.path.join(ROOT, "cases")


def struct_hash(m: O.Csr) -> str:
    h = hashlib.sha256()
    h.update(np.asarray([m.rows, m.cols], np.int64).tobytes())
    h.update(np.ascontiguousarray(m.rp, np.int32).tobytes())
    h.update(np.ascontiguousarray(m.ci, np.int32).tobytes())
    return h.hexdigest()


def value_hash(m: O.Csr) -> str:
    return hashlib.sha256(np.ascontiguousarray(m.v, np.float64).tobytes()).hexdigest()


def mat_summary(m: O.Csr) -> dict:
    return dict(rows=m.rows, cols=m.cols, nnz=m.nnz, struct=struct_hash(m), values=value_hash(m),
                vsum=float(np.sum(m.v)), vabs=float(np.sum(np.abs(m.v))))


def bench_rhs(A: O.Csr, pin=0):
    """runner.hpp:184-189: b = A w, w_i = sin(0.7 i + 0.3), w[pin] = 0, unit norm."""
    w = np.sin(0.7 * np.arange(A.rows) + 0.3)
    w[pin] = 0.0
    w /= np.sqrt(np.dot(w, w))
    return O.ref().spmv(A, w)


def case_summary(R, name, h_min=0.0, dt=0.0, steps=2):
    c = R.case(os.path.join(CASES, name + ".cfg"), h_min, dt)
    out = dict(nx=c.nx, ny=c.ny, n_q=c.n_q, n_p=c.n_p, n_b=c.n_b, n_lambda=c.n_lambda, h_min=h_min, dt=dt)
    for k in ("G", "E", "H", "A", "BN", "Q", "QT", "lhs2"):
        out[k] = mat_summary(c.op(k))
    h = c.hierarchy()
    lv = []
    L2 = c.op("lhs2")
    A = L2
    for l in range(h.n_levels):
        d = h.level(l)
        n_core = d["A"].rows - 2 * c.n_b
        theta = 0.25 * 0.5 ** l
        n_agg, agg = R.aggregate(d["A"], theta, n_core)
        lv.append(dict(A=mat_summary(d["A"]), P=mat_summary(d["P"]), Pt=mat_summary(d["Pt"]), omega=d["omega"],
                       n_agg=n_agg, agg=hashlib.sha256(np.ascontiguousarray(agg, np.int32).tobytes()).hexdigest()))
    out["levels"] = lv
    out["coarse"] = mat_summary(h.coarse())
    out["stalled"] = h.stalled
    b = bench_rhs(L2)
    r = R.pcg(L2, b, None, kind=2, hier=h)
    out["bench_pcg_sa"] = dict(iterations=r["iterations"], rel_residual=r["rel_residual"])
    rd = R.pcg(L2, b, None, kind=1)
    out["bench_pcg_diag"] = dict(iterations=rd["iterations"], rel_residual=rd["rel_residual"])
    st = []
    for _ in range(steps):
        rep = c.step()
        f = c.forces() if c.n_b else dict(cd=0.0, cl=0.0)
        st.append(dict(s1=int(rep["solve1_iters"]), s2=int(rep["solve2_iters"]), div=rep["div_residual"],
                       slip=rep["noslip_residual"], cd=f["cd"], cl=f["cl"],
                       qn=float(np.linalg.norm(c.state("q"))), ln=float(np.linalg.norm(c.state("lambda")))))
    out["steps"] = st
    return out


def main():
    R = O.ref()
    hashes = {}
    for name, hm in (("cavity", 0.0), ("cylinder_re40_smoke", 0.0), ("flapping_smoke", 0.0), ("cylinder_re40", 0.0)):
        print("case", name, flush=True)
        hashes[name] = case_summary(R, name, hm)
    print("case uniform_cylinder N=256", flush=True)
    hashes["uniform_cylinder_256"] = case_summary(R, "uniform_cylinder", 30.72 / 256, 0.06)
    # synthetic fixtures (proj/tests/oracles.hpp)
    for n in (8, 20, 64):
        A = O.poisson5(n)
        h = R.sa_build(A)
        hashes[f"poisson5_{n}"] = dict(
            levels=[dict(A=mat_summary(h.level(l)["A"]), P=mat_summary(h.level(l)["P"]), omega=h.level(l)["omega"])
                    for l in range(h.n_levels)], coarse=mat_summary(h.coarse()))
    with open(os.path.join(HERE, "hashes.json"), "w") as f:
        json.dump(hashes, f, indent=1, sort_keys=True)

    # full small case
    c = R.case(os.path.join(CASES, "uniform_cylinder.cfg"), 30.72 / 64, 0.2)
    arrs = dict(dims=np.array([c.nx, c.ny, c.n_q, c.n_p, c.n_b, c.n_lambda]))
    g = c.grid()
    for k in O.RefCase.GRID:
        arrs["grid_" + k] = g[k]
    arrs["grid_uniform"] = g["uniform"]
    arrs["grid_h_min"] = np.array([g["h_min"]])
    bd = c.bodies()
    for k, v in bd.items():
        arrs["body_" + k] = v
    for k in ("G", "E", "H", "A", "BN", "Q", "QT", "lhs2"):
        m = c.op(k)
        arrs[k + "_rp"], arrs[k + "_ci"], arrs[k + "_v"] = m.rp, m.ci, m.v
        arrs[k + "_shape"] = np.array([m.rows, m.cols])
    h = c.hierarchy()
    arrs["n_levels"] = np.array([h.n_levels])
    for l in range(h.n_levels):
        d = h.level(l)
        for k in ("A", "P", "Pt"):
            arrs[f"L{l}_{k}_rp"], arrs[f"L{l}_{k}_ci"], arrs[f"L{l}_{k}_v"] = d[k].rp, d[k].ci, d[k].v
            arrs[f"L{l}_{k}_shape"] = np.array([d[k].rows, d[k].cols])
        arrs[f"L{l}_omega"] = np.array([d["omega"]])
        n_agg, agg = R.aggregate(d["A"], 0.25 * 0.5 ** l, d["A"].rows - 2 * c.n_b)
        arrs[f"L{l}_agg"] = agg
    b = bench_rhs(c.op("lhs2"))
    arrs["bench_b"] = b
    r = R.pcg(c.op("lhs2"), b, None, kind=2, hier=h, history=True)
    arrs["bench_x"], arrs["bench_hist"] = r["x"], r["history"]
    arrs["bench_iters"] = np.array([r["iterations"]])
    arrs["vcycle_z"] = h.apply(b)
    for s in range(3):
        rep = c.step()
        arrs[f"step{s}_q"] = c.state("q")
        arrs[f"step{s}_lambda"] = c.state("lambda")
        arrs[f"step{s}_iters"] = np.array([rep["solve1_iters"], rep["solve2_iters"]])
        f = c.forces()
        arrs[f"step{s}_forces"] = np.array([f["fx"], f["fy"], f["cd"], f["cl"]])
    np.savez_compressed(os.path.join(HERE, "small_case.npz"), **arrs)
    print("done")


if __name__ == "__main__":
    main()
