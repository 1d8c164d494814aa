"""Full-size golden hashes from the unmodified reference (oracle/_ref): C2 (1042^2) and S-4M
(2040^2). Structure hashes of E, H, lhs2 and every SA level's A/P, omegas, aggregate hashes and
the first step's iteration counts / Cd. Slow (S-4M setup ~2 min): run once in the build
container:  python tests/golden/make_golden_large.py"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402
from tests.golden.make_golden import case_summary  # noqa: E402

R = O.ref()
R.set_threads(os.cpu_count() or 1)
out = {}
for key, (name, h, dt) in {"c2": ("cylinder_re40", 0.002, 0.001), "s4m": ("cylinder_re3000", 0.001, 2.5e-4)}.items():
    print(key, flush=True)
    out[key] = case_summary(R, name, h, dt, steps=1)
with open(os.path.join(HERE, "hashes_large.json"), "w") as f:
    json.dump(out, f, indent=1, sort_keys=True)
print("done")
