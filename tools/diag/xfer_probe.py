"""Level-0 stencil transfers (xfer.cuh) vs the explicit P / P^T on the same hierarchy: eligibility,
V-cycle difference, PCG iterations.  python tools/diag/xfer_probe.py c2 s4m"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import bench
from paper_1109_3524_b200 import ibm

for wl in sys.argv[1:]:
    if wl.endswith(".cfg"):
        st = ibm.Stepper(wl)
    else:
        cfg, h, dt, _ = bench.workload(wl)
        st = ibm.Stepper(os.path.join("cases", cfg + ".cfg"), h_min=h, dt=dt)
    hh = st.hierarchy()
    A = hh.level(0)["A"]
    n = A.rows()
    rng = np.random.default_rng(3)
    r = rng.uniform(-1, 1, n)
    on = hh.transfers(1)
    z1 = ibm.sa_apply(hh, r)
    hh.transfers(0)
    z0 = ibm.sa_apply(hh, r)
    rel = np.max(np.abs(z1 - z0)) / np.max(np.abs(z0))
    p = ibm.SolverParams(rel_tol=1e-8, max_iters=2000)
    r0 = ibm.pcg(A, r, None, ibm.SaPreconditioner(hh), p)
    hh.transfers(1)
    r1 = ibm.pcg(A, r, None, ibm.SaPreconditioner(hh), p)
    xr = np.max(np.abs(r1.x - r0.x)) / np.max(np.abs(r0.x))
    print(wl, "rows", n, "on", on, "vcycle rel diff %.3e" % rel, "pcg its", r0.iterations, r1.iterations,
          "x rel %.2e" % xr, flush=True)
