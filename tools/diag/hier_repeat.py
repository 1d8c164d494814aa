"""Build the SA hierarchy of a case's lhs2 several times; report which level/matrix differs."""
import os, sys, hashlib
sys.path.insert(0, os.getcwd())
import numpy as np
import bench
from paper_1109_3524_b200 import ibm
from tests import helpers as H
wl = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg, h_min, dt, _ = bench.workload(wl)
st = ibm.Stepper(os.path.join("cases", cfg + ".cfg"), h_min=h_min, dt=dt)
A = st.op("lhs2")
def dig(h):
    out = []
    for l in range(h.n_levels):
        lv = h.level(l)
        row = []
        for k in ("A", "P", "Pt"):
            rp, ci, v = lv[k].csr()
            row.append(hashlib.sha1(rp.tobytes() + ci.tobytes()).hexdigest()[:6] + "/" + hashlib.sha1(v.tobytes()).hexdigest()[:6])
        na, agg = h.aggregates(l)
        row.append("om%.17g" % lv["omega"])
        row.append("agg" + hashlib.sha1(agg[:lv["A"].rows()].tobytes()).hexdigest()[:6])
        out.append(row)
    return out
ref = None
for k in range(n):
    hh = ibm.build_sa_hierarchy(A, ibm.SaOptions(keep_fine_tail=2 * st.n_b))
    d = dig(hh)
    if ref is None:
        ref = d
    diffs = [(l, j) for l in range(min(len(d), len(ref))) for j in range(5) if d[l][j] != ref[l][j]]
    print(os.environ.get("TAG", ""), wl, k, "levels", len(d), "diffs", diffs[:8], flush=True)
    ibm.spmm(A, A)
