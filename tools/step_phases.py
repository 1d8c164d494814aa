"""Per-phase wall time of Stepper.advance (StepReport's PhaseTimes, stepper.hpp:139-144).

  python tools/step_phases.py [--workload flapping] [--steps 10] [--warmup 3]

Prints one JSON line: mean seconds per step of each phase, how often the operators and the
SA hierarchy were rebuilt, and the mean solve iteration counts. Used to find where a
moving-body step goes (refresh of E/H/Q/lhs2 every step, SA rebuild every n_pc steps).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1109_3524_b200 import ibm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="flapping")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    cfg, h_min, dt, _ = bench.workload(a.workload)
    st = ibm.Stepper(os.path.join(bench.CASES, cfg + ".cfg"), h_min=h_min, dt=dt)
    for _ in range(a.warmup):
        st.advance()
    keys = ("t_assembly", "t_precond", "t_explicit", "t_solve1", "t_solve2", "t_projection")
    tot = dict.fromkeys(keys, 0.0)
    n_ops = n_hier = it1 = it2 = 0
    for _ in range(a.steps):
        r = st.advance()
        assert r.ok, r.message
        for k in keys:
            tot[k] += getattr(r, k)
        n_ops += r.rebuilt_operators
        n_hier += r.rebuilt_hierarchy
        it1 += r.solve1_iters
        it2 += r.solve2_iters
    out = {k: round(v / a.steps * 1e3, 3) for k, v in tot.items()}
    out.update(unit="ms per step", workload=a.workload, steps=a.steps, operator_rebuilds=n_ops,
               hierarchy_rebuilds=n_hier, solve1_iters=it1 / a.steps, solve2_iters=it2 / a.steps)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
