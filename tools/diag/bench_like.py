"""Mimic bench.run_ours step by step with per-step status (flaky solve hunt)."""
import os, sys
sys.path.insert(0, os.getcwd())
import bench
from paper_1109_3524_b200 import ibm
wl = sys.argv[1]; mode = sys.argv[2]; n = int(sys.argv[3])
cfg, h, dt, _ = bench.workload(wl)
ctx = ibm.Context(0)
st = ibm.Stepper(os.path.join("cases", cfg + ".cfg"), h_min=h, dt=dt, ctx=ctx)
if "hier" in mode:
    bench.hier_bytes(st.hierarchy())
if "ops" in mode:
    A = st.op("A"); Lm, QT, Q, BN = st.op("L"), st.op("QT"), st.op("Q"), st.op("BN")
for k in range(n):
    if "timer" in mode:
        ctx.timer_start()
    r = st.advance()
    if "timer" in mode:
        ctx.timer_stop()
    if "forces" in mode:
        st.forces(); st.get("f_tilde"); st.phase_ms()
    print(wl, mode, k, r.ok, r.message, r.solve1_iters, r.solve2_iters, "%.3e %.3e" % (r.solve1_res, r.solve2_res), flush=True)
    if not r.ok:
        break
