"""Cost of the row-slab decomposition on one GPU (csrc/dist.cu, loopback communicator).

For a workload's coupled system (bench_rhs of runner.hpp) it times, on the device:
  single   ibmgpu_pcg (one conditional-graph launch)
  dist R   ibmgpu_dist_pcg with R emulated ranks (one graph launch per iteration, halos by D2D copy)
Loopback runs every rank's kernels back to back on this GPU, so time/R approximates one rank's
compute share when the R slabs run on R GPUs (communication not included; the loopback halo copies
are). b and x stay on the device; nothing crosses PCIe inside the timed region. Prints JSON.

  python tools/dist_bench.py [--workload c2|s4m|c5-N] [--ranks 1,2,4,8] [--min-dist-rows 200000]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CASES, workload  # noqa: E402
from paper_1109_3524_b200 import ibm  # noqa: E402


def cell_j(y_faces, y):
    return np.clip(np.searchsorted(y_faces, y, side="right") - 1, 0, len(y_faces) - 2).astype(np.int32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--min-dist-rows", type=int, default=200000)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--iters", type=int, default=0, help="force exactly this many iterations (timing only)")
    ap.add_argument("--nccl", action="store_true",
                    help="one-rank NCCL communicator: the R virtual ranks' halos go through ncclSend/ncclRecv "
                         "to self and every allreduce through ncclAllReduce (captured in the iteration graph)")
    a = ap.parse_args()
    cfg, h_min, dt, desc = workload(a.workload)
    kw = {}
    if a.nccl:
        kw["ctx"] = ibm.Context(0, nranks=1, rank=0, nccl_id=ibm.nccl_unique_id())
    st = ibm.Stepper(os.path.join(CASES, cfg + ".cfg"), h_min=h_min, dt=dt, **kw)
    ctx = st.ctx
    A = st.op("lhs2")
    n = A.rows()
    w = np.sin(0.7 * np.arange(n) + 0.3)
    w[0] = 0.0
    w /= np.linalg.norm(w)
    b = A.spmv(w)
    M = ibm.SaPreconditioner(st.hierarchy())
    bd = ibm.DeviceVector.from_host(b, ctx)
    out = {"workload": a.workload, "desc": desc, "n": n, "nccl": a.nccl, "results": []}

    def timed(fn):
        fn()
        best = 1e30
        res = None
        for _ in range(a.reps):
            ctx.sync()
            ctx.timer_start()
            res = fn()
            best = min(best, ctx.timer_stop())
        return best, res

    import ctypes as C
    from paper_1109_3524_b200._lib import SolveResultC
    lib = ctx.lib
    pc = (ibm.SolverParams(rel_tol=1e-30, max_iters=a.iters) if a.iters else ibm.SolverParams()).c()

    # Device-resident solves: b stays on the device; x0 = 0 is a fresh device allocation (device
    # memset); no host transfer inside the timed region.
    def single():
        x = ibm.DeviceVector(n, ctx)
        res = SolveResultC()
        ctx.check(lib.ibmgpu_pcg(ctx.h, A.h, M.kind, M.hier.h, bd.p, x.p, C.byref(pc), C.byref(res), None))
        return res

    ms, r = timed(single)
    out["results"].append({"mode": "single", "ms": round(ms, 3), "iters": r.iterations,
                           "ms_per_iter": round(ms / r.iterations, 4)})
    yf, by = st.grid()["y_faces"], st.bodies()["y"]
    for R in (int(x) for x in a.ranks.split(",")):
        owner = ibm.partition_lambda(st.nx, st.ny, cell_j(yf, by), R)
        t0 = time.time()
        ds = ibm.DistSolver(A, M, owner, virtual_ranks=R, min_dist_rows=a.min_dist_rows)
        setup = time.time() - t0
        def dist_solve():
            x = ibm.DeviceVector(n, ctx)
            res = SolveResultC()
            ctx.check(lib.ibmgpu_dist_pcg(ds.h, bd.p, x.p, C.byref(pc), C.byref(res), None))
            return res

        ms, r = timed(dist_solve)
        info = ds.info()
        out["results"].append({"mode": f"{'nccl-self' if a.nccl else 'loopback'} R={R}", "backend": info["loopback"], "ms": round(ms, 3), "iters": r.iterations,
                               "ms_per_iter": round(ms / r.iterations, 4),
                               "per_rank_ms_per_iter": round(ms / r.iterations / R, 4),
                               "dist_levels": info["dist_levels"], "levels": info["levels"],
                               "rank0_own": info["own_rows"], "rank0_halo": info["halo"],
                               "setup_s": round(setup, 2)})
        del ds
    print(json.dumps(out))


if __name__ == "__main__":
    main()
