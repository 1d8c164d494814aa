import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1109_3524_b200 import ibm
cfg, h, dt, n = sys.argv[1], float(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
st = ibm.Stepper(os.path.join("cases", cfg + ".cfg"), h_min=h, dt=dt)
out = []
for s in range(n):
    r = st.advance()
    if not r.ok:
        out.append(f"{s}:FAIL"); break
    if s % 5 == 4 or s < 3:
        q = st.get("q")
        out.append("%d:%.3g/%d" % (s, np.max(np.abs(q)), r.solve2_iters))
print(cfg, h, dt, " ".join(out), flush=True)
