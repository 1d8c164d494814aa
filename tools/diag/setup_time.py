import sys, os, time
sys.path.insert(0, os.getcwd())
t00 = time.time()
import bench
from paper_1109_3524_b200 import ibm
wl = sys.argv[1]
cfg, h, dt, _ = bench.workload(wl)
t0 = time.time()
ctx = ibm.Context.default()
t1 = time.time()
st = ibm.Stepper(os.path.join("cases", cfg + ".cfg"), h_min=h, dt=dt, ctx=ctx)
t2 = time.time()
r = st.advance()
st.ctx.sync()
t3 = time.time()
print(wl, os.environ.get("IBMGPU_POOL_RESERVE_MB"), "import %.2f ctx %.2f stepper %.2f first step %.2f  time-to-first-step %.2f" % (t0 - t00, t1 - t0, t2 - t1, t3 - t2, t3 - t0), flush=True)
