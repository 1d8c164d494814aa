import sys, os
sys.path.insert(0, os.getcwd())
from paper_1109_3524_b200 import ibm
wl = sys.argv[1]
import bench
cfg, h, dt, _ = bench.workload(wl)
ctx = ibm.Context(0) if sys.argv[2] == "explicit" else ibm.Context.default()
st = ibm.Stepper(os.path.join("cases", cfg + ".cfg"), h_min=h, dt=dt, ctx=ctx)
for k in range(int(os.environ.get("STEPS", "6"))):
    r = st.advance()
    print(wl, sys.argv[2], os.environ.get("IBMGPU_POOL_RESERVE_MB"), k, r.ok, r.message, r.solve1_iters, r.solve2_iters, flush=True)
