"""flapping.cfg throughput and the per-phase host-side wait/solve times of Stepper::advance
(IBMGPU_SETUP_PROFILE=1 additionally prints the setup laps on stderr)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_1109_3524_b200 import ibm
st = ibm.Stepper(sys.argv[2] if len(sys.argv) > 2 else "cases/flapping.cfg")
for _ in range(4):
    st.advance()
st.ctx.sync()
t = time.time()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
acc = {}
its = 0
for _ in range(n):
    r = st.advance()
    its += r.solve2_iters
    for k in ("t_assembly", "t_precond", "t_explicit", "t_solve1", "t_solve2", "t_projection"):
        acc[k] = acc.get(k, 0.0) + getattr(r, k)
st.ctx.sync()
dt = time.time() - t
print("steps/s %.2f  cg its/step %.1f  ms/step %.2f | " % (n / dt, its / n, 1e3 * dt / n) +
      " ".join("%s %.2f ms" % (k[2:], 1e3 * v / n) for k, v in acc.items()), file=sys.stderr)
