"""BASELINE metric "CG iters/sec vs grid size; SpMV HBM GB/s vs 8 TB/s" on the synthetic uniform
cylinder grids (BASELINE configs[4], C5-N: N^2 cells): for each N, one SA-PCG solve of the coupled
system on the runner.hpp bench right-hand side (device-resident b and x) and a timed lhs2 SpMV,
plus two Stepper::advance steps (steps/s). One JSON line per grid.

  python tools/sweep.py --sizes 1024,2048,4096,8192
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1109_3524_b200 import ibm  # noqa: E402
from paper_1109_3524_b200._lib import SolveResultC  # noqa: E402


def sweep(sizes, spmv_reps=20, emit=None):
    """One record per C5-N grid (see module doc); emit(record) is called as each finishes."""
    peak, kind = bench.load_peaks()
    out = []
    for N in sizes:
        cfg, h, dt, desc = bench.workload(f"c5-{N}")
        t0 = time.time()
        st = ibm.Stepper(os.path.join(ROOT, "cases", cfg + ".cfg"), h_min=h, dt=dt)
        setup = time.time() - t0
        ctx, A = st.ctx, st.op("lhs2")
        n = A.rows()
        w = np.sin(0.7 * np.arange(n) + 0.3)
        w[0] = 0.0
        w /= np.linalg.norm(w)
        b = ibm.DeviceVector.from_host(A.spmv(w), ctx)
        M = ibm.SaPreconditioner(st.hierarchy())
        pc = ibm.SolverParams().c()

        def solve():
            x = ibm.DeviceVector(n, ctx)
            res = SolveResultC()
            ctx.check(ctx.lib.ibmgpu_pcg(ctx.h, A.h, M.kind, M.hier.h, b.p, x.p, C.byref(pc), C.byref(res), None))
            return res

        solve()
        ctx.sync()
        ctx.timer_start()
        r = solve()
        ms = ctx.timer_stop()
        b_it2, _ = bench.hier_bytes(st.hierarchy())
        x = ibm.DeviceVector(n, ctx)
        y = ibm.DeviceVector(n, ctx)
        A.spmv_into(x, y)
        ctx.sync()
        ctx.timer_start()
        for _ in range(spmv_reps):
            A.spmv_into(x, y)
        spmv_ms = ctx.timer_stop() / spmv_reps
        sb = bench.spmv_bytes(n, n, A.nnz())  # reference-CSR (algorithmic) bytes
        fb, _ = A.format_bytes()  # bytes the stencil/DIA format actually streams
        st.advance()
        ctx.sync()
        ctx.timer_start()
        reps = [st.advance() for _ in range(2)]
        step_ms = ctx.timer_stop() / 2
        it_ms = ms / max(r.iterations, 1)
        rec = {
            "grid": f"{N}^2", "cells": N * N, "n_lambda": n, "nnz_lhs2": A.nnz(), "setup_s": round(setup, 2),
            "cg_iters": r.iterations, "cg_iteration_ms": round(it_ms, 4),
            "cg_iters_per_s": round(1e3 / it_ms, 1),
            "cg_hbm_gbs": round(b_it2 / (it_ms * 1e-3) / 1e9, 1), "cg_frac_measured": round(b_it2 / (it_ms * 1e-3) / 1e9 / peak, 4),
            "spmv_lhs2_us": round(spmv_ms * 1e3, 1),
            # roofline of the SpMV on the bytes its format moves (no column indices in the band)
            "spmv_format_gbs": round(fb / (spmv_ms * 1e-3) / 1e9, 1),
            # (a read-dominated stream can exceed the copy-measured peak, which pays for writes)
            "spmv_format_frac_measured": round(fb / (spmv_ms * 1e-3) / 1e9 / peak, 4),
            "spmv_format_frac_of_8tbs": round(fb / (spmv_ms * 1e-3) / 8e12, 4),
            # reference-CSR bytes (12/nnz) per second: a CSR-equivalent rate, not a roofline fraction
            "spmv_csr_equiv_gbs": round(sb / (spmv_ms * 1e-3) / 1e9, 1),
            "steps_per_s": round(1e3 / step_ms, 3), "solve2_iters_per_step": [rr.solve2_iters for rr in reps],
            "peak_kind": kind}
        out.append(rec)
        if emit:
            emit(rec)
        del st
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1024,2048,4096,8192")
    ap.add_argument("--spmv-reps", type=int, default=20)
    a = ap.parse_args()
    sweep([int(s) for s in a.sizes.split(",")], a.spmv_reps, emit=lambda r: print(json.dumps(r), flush=True))


if __name__ == "__main__":
    main()
