import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import bench
from oracle import oracle as O
cfg, h, dt, _ = bench.workload(sys.argv[1] if len(sys.argv) > 1 else "s4m")
R = O.ref(); R.set_threads(os.cpu_count())
t0 = time.time()
c = R.case(os.path.join("cases", cfg + ".cfg"), h, dt)
print("setup", time.time() - t0, flush=True)
for k in range(int(sys.argv[2]) if len(sys.argv) > 2 else 7):
    r = c.step()
    q = c.state("q")
    print(k, bool(r["ok"]), int(r["solve1_iters"]), int(r["solve2_iters"]), "qmax %.4e" % np.max(np.abs(q)), "%.1fs" % (time.time() - t0), flush=True)
