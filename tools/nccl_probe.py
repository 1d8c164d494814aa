"""Exercise the NCCL backend plumbing on whatever GPUs are visible: rank 0 makes the id
(ibmgpu_nccl_unique_id), ranks init contexts (ibmgpu_init with nranks>1) and, if that succeeds,
run one distributed C2a solve (ibmgpu_stepper_distribute) and compare with a single-GPU solve.
With fewer GPUs than ranks every rank uses device rank % ngpus (NCCL normally refuses two ranks on
one device; the probe then reports that cleanly instead of hanging).

  python tools/nccl_probe.py --ranks 2
"""
import argparse
import json
import multiprocessing as mp
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, R, uid, q):
    try:
        import numpy as np
        from paper_1109_3524_b200 import ibm
        ngpu = int(os.environ.get("PROBE_NGPU", "1"))
        ctx = ibm.Context(rank % ngpu, nranks=R, rank=rank, nccl_id=uid)
        st = ibm.Stepper(os.path.join(ROOT, "cases", "cylinder_re40.cfg"), ctx=ctx)
        st.distribute(min_dist_rows=0)
        rep = st.advance()
        q.put((rank, "ok", rep.ok, rep.solve2_iters, float(np.linalg.norm(st.get("lambda")))))
    except Exception as e:
        q.put((rank, "error", repr(e)[:300], -1, 0.0))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, default=2)
    a = ap.parse_args()
    from paper_1109_3524_b200 import ibm
    uid = ibm.nccl_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, a.ranks, uid, q)) for r in range(a.ranks)]
    for p in ps:
        p.start()
    out = []
    for _ in ps:
        try:
            out.append(q.get(timeout=120))
        except Exception:
            out.append((-1, "timeout", "", -1, 0.0))
    for p in ps:
        p.join(timeout=5)
        if p.is_alive():
            p.kill()
    print(json.dumps({"uid_bytes": len(uid), "results": sorted(out)}))


if __name__ == "__main__":
    main()
