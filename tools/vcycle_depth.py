"""In-graph cost of each SA level inside the real solve: SA-PCG on the workload's coupled system
for a fixed number of iterations, with the V-cycle truncated after k levels
(IBMGPU_DEBUG_VDEPTH=k, timing only: results are wrong) for k = 1..L, and the full cycle
(k = L+1, with the coarse solve). The difference between consecutive depths is the level's
marginal cost per iteration, with the real working set streaming through L2 (unlike the
back-to-back figures of tools/level_spmv.py).

  python tools/vcycle_depth.py --workload c2 [--iters 60]
"""
import argparse
import ctypes as C
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(workload, iters):
    import bench
    from paper_1109_3524_b200 import ibm
    from paper_1109_3524_b200._lib import SolveResultC
    cfg, h_min, dt, _ = bench.workload(workload)
    st = ibm.Stepper(os.path.join(ROOT, "cases", cfg + ".cfg"), h_min=h_min, dt=dt)
    ctx, A = st.ctx, st.op("lhs2")
    n = A.rows()
    b = ibm.DeviceVector.from_host(np.sin(0.7 * np.arange(n) + 0.3), ctx)
    M = ibm.SaPreconditioner(st.hierarchy())
    pc = ibm.SolverParams(rel_tol=1e-30, max_iters=iters).c()

    def solve():
        x = ibm.DeviceVector(n, ctx)
        res = SolveResultC()
        ctx.check(ctx.lib.ibmgpu_pcg(ctx.h, A.h, M.kind, M.hier.h, b.p, x.p, C.byref(pc), C.byref(res), None))
        return res

    solve()
    best = 1e30
    for _ in range(3):
        ctx.sync()
        ctx.timer_start()
        r = solve()
        best = min(best, ctx.timer_stop())
    return {"levels": st.hierarchy().n_levels, "iters": r.iterations, "ms_per_iter": round(best / max(r.iterations, 1), 4)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--iters", type=int, default=60)
    ap.add_argument("--depth", type=int, default=-1, help=argparse.SUPPRESS)
    a = ap.parse_args()
    if a.depth >= 0:
        print(json.dumps(one(a.workload, a.iters)))
        return
    out, L, k = [], None, 1
    while L is None or k <= L + 1:
        env = dict(os.environ, IBMGPU_DEBUG_VDEPTH=str(k))
        p = subprocess.run([sys.executable, __file__, "--workload", a.workload, "--iters", str(a.iters), "--depth", str(k)],
                           env=env, capture_output=True, text=True, check=True)
        rec = json.loads(p.stdout.strip().splitlines()[-1])
        L = rec["levels"]
        rec["depth"] = k
        if out:
            rec["marginal_us"] = round(1e3 * (rec["ms_per_iter"] - out[-1]["ms_per_iter"]), 1)
        out.append(rec)
        print(json.dumps(rec), flush=True)
        k += 1


if __name__ == "__main__":
    main()
