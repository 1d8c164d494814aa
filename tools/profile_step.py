"""Profile one Stepper::advance of a workload: warm-up steps, then cuProfilerStart / one step /
cuProfilerStop, so `ncu --profile-from-start off` captures exactly the kernels of one step.

  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file launches.csv python tools/profile_step.py --workload s4m
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT))
import bench  # noqa: E402
from paper_1109_3524_b200 import ibm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="s4m")
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--steps", type=int, default=1)
a = ap.parse_args()
cfg, h, dt, _ = bench.workload(a.workload)
st = ibm.Stepper(os.path.join(ROOT, "cases", cfg + ".cfg"), h_min=h, dt=dt)
for _ in range(a.warmup):
    st.advance()
cuda = ctypes.CDLL("libcuda.so.1")
st.ctx.sync()
cuda.cuProfilerStart()
for _ in range(a.steps):
    r = st.advance()
st.ctx.sync()
cuda.cuProfilerStop()
print(f"step ok={r.ok} s1={r.solve1_iters} s2={r.solve2_iters} phases={st.phase_ms()}")
