import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import bench
from paper_1109_3524_b200 import ibm
cfg, h, dt, _ = bench.workload("s4m")
st = ibm.Stepper(os.path.join("cases", cfg + ".cfg"), h_min=h, dt=dt)
def stats(tag):
    out = [tag]
    for k in ("q", "lambda", "conv_prev", "boundary"):
        a = st.get(k)
        out.append("%s finite=%s max=%.3e" % (k, np.isfinite(a).all(), np.nanmax(np.abs(a))))
    print(" | ".join(out), flush=True)
for k in range(12):
    r = st.advance()
    print(k, r.ok, r.message, r.solve1_iters, r.solve2_iters, r.bc_cfl, flush=True)
    stats(f"after {k}")
    if not r.ok:
        break
b = st.get("boundary")
nx, ny = st.nx, st.ny
names = ["left_u", "right_u", "left_v", "right_v", "bottom_v", "top_v", "bottom_u", "top_u"]
sizes = [ny, ny, ny - 1, ny - 1, nx, nx, nx - 1, nx - 1]
o = 0
for nme, n in zip(names, sizes):
    seg = b[o:o + n]; o += n
    print(nme, np.isfinite(seg).all(), seg.min(), seg.max())
