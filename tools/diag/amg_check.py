import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1109_3524_b200 import ibm
from oracle import oracle as O
from tests import helpers as H
ref = O.ref()
for name in ("cylinder_re40_smoke", "flapping_smoke", "cylinder_re40"):
    st = ibm.Stepper(H.case(name))
    A = st.op("lhs2")
    b = H.bench_rhs(A.spmv, A.rows())
    h = ibm.build_sa_hierarchy(A, ibm.SaOptions(keep_fine_tail=2 * st.n_b))
    r = ibm.amg_solve(A, h, b, None, ibm.SolverParams(max_iters=300))
    nf, nd = h.folded()
    kinds = [h.level(l)["A"].format_bytes()[1] for l in range(h.n_levels)]
    print(os.environ.get("TAG"), name, "amg its", r.iterations, "res %.3e" % r.rel_residual, "status", r.status, "folded", nf, nd, "kinds", kinds, flush=True)
