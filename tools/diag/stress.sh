#!/bin/bash
# fresh-process repetition of the bench's warm-up on S-4M and C2 (flaky-NaN hunt); one line per run
OUT=${OUT:-gpurun_out/stress.log}
for rep in $(seq 1 ${REPS:-6}); do
  for w in s4m c2; do
    python tools/diag/nan_probe.py $w explicit 2>&1 | tail -n 3 | tr '\n' ' ' >> $OUT
    echo " [env ${TAG:-default}]" >> $OUT
  done
done
