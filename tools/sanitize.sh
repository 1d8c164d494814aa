#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over smoke() and two steps of
# flapping_smoke (moving body: refresh, SA rebuild, both solves). Logs to gpurun_out/.
#   gpurun -- bash tools/sanitize.sh
set -u
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
cat > /tmp/flap2.py <<'PY'
import sys; sys.path.insert(0, ".")
from paper_1109_3524_b200 import ibm
st = ibm.Stepper("cases/flapping_smoke.cfg")
for _ in range(2):
    r = st.advance(); assert r.ok, r.message
print("flapping_smoke 2 steps ok", r.solve2_iters)
PY
for tool in memcheck racecheck synccheck initcheck; do
  for prog in smoke flap2; do
    if [ $prog = smoke ]; then cmd="python -c 'import __graft_entry__ as g; g.smoke()'"; else cmd="python /tmp/flap2.py"; fi
    echo "== $tool $prog" > "$OUT/sanitizer_${tool}_${prog}.txt"
    eval timeout 900 $CS --tool $tool --error-exitcode 17 --print-limit 50 $cmd >> "$OUT/sanitizer_${tool}_${prog}.txt" 2>&1
    echo "rc=$?" >> "$OUT/sanitizer_${tool}_${prog}.txt"
  done
done
