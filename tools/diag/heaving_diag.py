"""Per-step iteration counts and field differences, device Stepper vs the reference, on a case.
  python tools/diag/heaving_diag.py <case> <steps> [extra cfg text]"""
import sys, os, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from oracle import oracle as O
from paper_1109_3524_b200 import ibm
from tests import helpers as H

name = sys.argv[1] if len(sys.argv) > 1 else "heaving"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
extra = sys.argv[3].replace("\\n", "\n") if len(sys.argv) > 3 else ""
path = H.case(name)
if extra:
    txt = open(path).read() + "\n" + extra + "\n"
    path = os.path.join(tempfile.mkdtemp(), name + ".cfg")
    open(path, "w").write(txt)
ref = O.ref()
rc = ref.case(path, 0.0, 0.0)
st = ibm.Stepper(path)
print("case", name, repr(extra), os.environ.get("IBMGPU_FOLD"))
for s in range(steps):
    a = rc.step(); r = st.advance()
    q, qr = st.get("q"), rc.state("q")
    lam, lr = st.get("lambda"), rc.state("lambda")
    n_p = st.n_p
    print(s, "it1", r.solve1_iters, int(a["solve1_iters"]), "it2", r.solve2_iters, int(a["solve2_iters"]),
          "res2 %.6e %.6e" % (r.solve2_res, a["solve2_res"]),
          "q %.2e phi %.2e f %.2e" % (H.rel_err(q, qr), H.rel_err(lam[:n_p], lr[:n_p]), H.rel_err(lam[n_p:], lr[n_p:])),
          "hier", r.rebuilt_hierarchy, flush=True)
