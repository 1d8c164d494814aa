"""Per-CG-iteration time of a workload (bench.case_probe) — run twice under different env
settings in one session for A/B comparisons:  python tools/ab_iter.py s4m c2"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workloads", nargs="+")
ap.add_argument("--steps", type=int, default=8)
a = ap.parse_args()
for w in a.workloads:
    r = bench.case_probe(argparse.Namespace(steps=a.steps), w)
    print(json.dumps({"workload": w, "tag": os.environ.get("TAG", ""), "cg_iteration_ms": r["cg_iteration_ms"],
                      "frac_measured": r["frac_measured"], "frac_of_8tbs": r["frac_of_8tbs"],
                      "steps_per_s": r["steps_per_s"], "cg_iters_per_step": r["cg_iters_per_step"]}), flush=True)
