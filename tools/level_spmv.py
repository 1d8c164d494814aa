"""Warm, in-graph time of every SpMV of a workload's SA hierarchy (A_l, P_l, P_lᵀ per level and
the lhs2 operator): `reps` back-to-back launches captured in one CUDA graph with programmatic
dependent launch (ibmgpu_spmv_timed), so the figure is the kernel's steady-state cost inside a
graph — unlike ncu's serialised, cache-flushed launch list. Algorithmic bytes per SURVEY §8(d).

  python tools/level_spmv.py --workload c2 [--reps 200]
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1109_3524_b200 import ibm  # noqa: E402


def timed(ctx, M, reps):
    x = ibm.DeviceVector.from_host(np.sin(np.arange(M.cols()) * 0.37), ctx)
    y = ibm.DeviceVector(M.rows(), ctx)
    us = C.c_double()
    ctx.check(ctx.lib.ibmgpu_spmv_timed(ctx.h, M.h, x.p, y.p, reps, C.byref(us)))
    return us.value


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--reps", type=int, default=200)
    a = ap.parse_args()
    cfg, h_min, dt, _ = bench.workload(a.workload)
    st = ibm.Stepper(os.path.join(ROOT, "cases", cfg + ".cfg"), h_min=h_min, dt=dt)
    ctx, h = st.ctx, st.hierarchy()
    total = 0.0
    for l in range(h.n_levels):
        lv = h.level(l)
        for k in ("A", "P", "Pt"):
            M = lv[k]
            us = timed(ctx, M, a.reps)
            b = bench.spmv_bytes(M.rows(), M.cols(), M.nnz())
            total += us * (2 if k == "A" else 1)
            print(json.dumps({"level": l, "op": k, "rows": M.rows(), "nnz": M.nnz(), "us": round(us, 2),
                              "gbs": round(b / (us * 1e-6) / 1e9, 1)}), flush=True)
    print(json.dumps({"sum_vcycle_spmv_us": round(total, 1)}))


if __name__ == "__main__":
    main()
