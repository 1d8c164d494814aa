import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import bench
from paper_1109_3524_b200 import ibm
wl = sys.argv[1] if len(sys.argv) > 1 else "s4m"
cfg, h, dt, _ = bench.workload(wl)
st = ibm.Stepper(os.path.join("cases", cfg + ".cfg"), h_min=h, dt=dt)
nx, ny = st.nx, st.ny
n_u = (nx - 1) * ny
g = st.grid()
def loc(k):
    if k < n_u:
        return "u i_f=%d j=%d x=%.4f y=%.4f" % (k % (nx - 1) + 1, k // (nx - 1), g["x_faces"][k % (nx - 1) + 1], g["y_c"][k // (nx - 1)])
    k -= n_u
    return "v i=%d j_f=%d x=%.4f y=%.4f" % (k % nx, k // nx + 1, g["x_c"][k % nx], g["y_faces"][k // nx + 1])
for s in range(int(sys.argv[2]) if len(sys.argv) > 2 else 7):
    r = st.advance()
    q = st.get("q")
    # velocity (q / transverse width)
    u = q.copy()
    dy = g["dy"]; dx = g["dx"]
    ju = np.arange(n_u) // (nx - 1)
    u[:n_u] /= dy[ju]
    iv = np.arange(len(q) - n_u) % nx
    u[n_u:] /= dx[iv]
    k = int(np.argmax(np.abs(u)))
    top = np.argsort(-np.abs(u))[:5]
    print(s, r.ok, r.solve1_iters, r.solve2_iters, "max|vel| %.4e at %s" % (abs(u[k]), loc(k)),
          "| top5:", "; ".join("%.3e %s" % (u[t], loc(int(t))) for t in top), flush=True)
