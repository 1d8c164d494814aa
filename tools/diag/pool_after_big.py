"""Moving-body throughput in a process that first ran a big static case (pool layout effect)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import bench
from paper_1109_3524_b200 import ibm
pre = sys.argv[1] if len(sys.argv) > 1 else "none"
if pre != "none":
    cfg, h, dt, _ = bench.workload(pre)
    st = ibm.Stepper(os.path.join("cases", cfg + ".cfg"), h_min=h, dt=dt)
    for _ in range(3):
        st.advance()
    st.ctx.sync()
    del st
st = ibm.Stepper("cases/flapping.cfg")
for _ in range(6):
    st.advance()
st.ctx.sync()
t = time.time()
w = 0.0
for _ in range(40):
    r = st.advance()
    w += r.t_assembly
st.ctx.sync()
print(pre, "steps/s %.1f wait %.2f ms" % (40 / (time.time() - t), 1e3 * w / 40), flush=True)
