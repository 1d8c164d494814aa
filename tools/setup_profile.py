"""Per-phase cost of the device SA hierarchy build (IBMGPU_SETUP_PROFILE=1 output on stderr):
builds the workload's stepper, then rebuilds the hierarchy of its lhs2 `--reps` times.

  IBMGPU_SETUP_PROFILE=1 python tools/setup_profile.py --workload flapping
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CASES, workload  # noqa: E402
from paper_1109_3524_b200 import ibm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="flapping")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
cfg, h_min, dt, _ = workload(a.workload)
st = ibm.Stepper(os.path.join(CASES, cfg + ".cfg"), h_min=h_min, dt=dt)
A = st.op("lhs2")
for _ in range(a.reps):
    st.ctx.sync()
    t = time.perf_counter()
    h = ibm.build_sa_hierarchy(A, ibm.SaOptions(keep_fine_tail=2 * st.n_b))
    st.ctx.sync()
    print(f"sa_build total {1e3 * (time.perf_counter() - t):.2f} ms, levels {h.n_levels}", file=sys.stderr, flush=True)
