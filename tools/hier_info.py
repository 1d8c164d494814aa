"""Per-level structure of a workload's SA hierarchy (rows, nnz, row-length profile), to relate
launch-list kernels to levels.  python tools/hier_info.py --workload c2"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CASES, workload  # noqa: E402
from paper_1109_3524_b200 import ibm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
a = ap.parse_args()
cfg, h_min, dt, _ = workload(a.workload)
st = ibm.Stepper(os.path.join(CASES, cfg + ".cfg"), h_min=h_min, dt=dt)
h = st.hierarchy()
for l in range(h.n_levels):
    lv = h.level(l)
    for k in ("A", "P", "Pt"):
        rp, _, _ = lv[k].csr()
        ln = np.diff(rp)
        print(f"L{l} {k:2s} rows {len(ln):8d} nnz {int(rp[-1]):9d} mean {ln.mean():6.1f} max {ln.max():5d} "
              f">96 {(ln > 96).sum():6d} ({100 * ln[ln > 96].sum() / max(rp[-1], 1):4.1f}% nnz)")
print("coarse n_c", h.info()[2])
