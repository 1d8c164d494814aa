"""First difference between the grid pass-1 aggregation and the LFMIS one on a case's level 0."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from tests.test_gpu_agg_grid import _agg, _planned
from oracle import oracle as O
from tests import helpers as H
from paper_1109_3524_b200 import ibm
name = sys.argv[1] if len(sys.argv) > 1 else "cylinder_re40_smoke"
st = ibm.Stepper(H.case(name))
A = st.op("lhs2")
rp, ci, v = A.csr()
Ah = O.Csr(A.rows(), A.cols(), rp, ci, v)
n_b = st.n_lambda - st.nx * st.ny if hasattr(st, "n_lambda") else 0
n_core = st.nx * st.ny
Ad = _planned(Ah)
print("rows", A.rows(), "n_core", n_core, "nx", st.nx, "ny", st.ny, "kind", Ad.format_bytes()[1])
res = {}
for k in ("grid", "lfmis"):
    os.environ["IBMGPU_AGG"] = k
    res[k] = _agg(Ad, 0.25, n_core)
print("n", res["grid"][0], res["lfmis"][0])
a, b = res["grid"][1], res["lfmis"][1]
d = np.nonzero(a != b)[0]
print("differ", len(d), d[:10], [(i // st.nx, i % st.nx) for i in d[:5]])
port = O.port()
n_ref, agg_ref = port.aggregate(Ah, 0.25, n_core)
print("oracle n", n_ref, "grid==oracle", np.array_equal(a, np.asarray(agg_ref)[:n_core]), "lfmis==oracle",
      np.array_equal(b, np.asarray(agg_ref)[:n_core]))
