#!/bin/bash
# A/B timing of library variants in one gpurun session (S-4M and C2 ms per CG iteration).
# Build each variant and copy it to abtest/lib_<name>.so (not gpurun-ignored), then:
#   gpurun -- bash tools/ab_run.sh base variant1 base ; cat gpurun_out/ab_results.txt
for v in "$@"; do
  IBMGPU_LIB=$PWD/abtest/lib_$v.so python bench.py --workload s4m --steps 3 --warmup 3 --no-cpu > gpurun_out/ab_s4m_$v.json 2>/dev/null
  IBMGPU_LIB=$PWD/abtest/lib_$v.so python bench.py --steps 10 --warmup 3 --no-cpu --no-s4m > gpurun_out/ab_c2_$v.json 2>/dev/null
  python -c "
import json
a=json.load(open('gpurun_out/ab_s4m_$v.json')); b=json.load(open('gpurun_out/ab_c2_$v.json')); print('$v', a['cg_iteration_ms'], b['cg_iteration_ms'])" >> gpurun_out/ab_results.txt
done
