"""Time plain SpMV (ibmgpu_spmv) on a workload's operators: algorithmic GB/s per matrix.
  python tools/spmv_bench.py --workload s4m"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1109_3524_b200 import ibm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="s4m")
ap.add_argument("--reps", type=int, default=50)
a = ap.parse_args()
cfg, h, dt, _ = bench.workload(a.workload)
st = ibm.Stepper(os.path.join(ROOT, "cases", cfg + ".cfg"), h_min=h, dt=dt)
hier = st.hierarchy()
mats = [("lhs2", st.op("lhs2")), ("A", st.op("A")), ("QT", st.op("QT")), ("Q", st.op("Q"))]
for l in range(hier.n_levels):
    lv = hier.level(l)
    mats += [(f"L{l}.A", lv["A"]), (f"L{l}.P", lv["P"]), (f"L{l}.Pt", lv["Pt"])]
ctx = st.ctx
for name, M in mats:
    x = ibm.DeviceVector(M.cols(), ctx)
    y = ibm.DeviceVector(M.rows(), ctx)
    for _ in range(3):
        M.spmv_into(x, y)
    ctx.sync()
    ctx.timer_start()
    for _ in range(a.reps):
        M.spmv_into(x, y)
    ms = ctx.timer_stop() / a.reps
    b = bench.spmv_bytes(M.rows(), M.cols(), M.nnz())
    print(f"{name:8s} rows {M.rows():9d} nnz {M.nnz():10d} {ms*1e3:9.1f} us  {b/ms/1e6:8.0f} GB/s (algorithmic)")
