#!/bin/bash
# Round-2 profile set (B200_PROFILING.md recipe; run each program once without ncu first):
#  1. ncu launch list (durations) of one S-4M and one C2 step
#  2. DRAM traffic of complete solve-2 iterations (S-4M, C2)
#  3. ncu --set full of ten solve-2 SpMV launches of an S-4M step
set -u
O=gpurun_out/r02prof
mkdir -p $O
python tools/profile_step.py --workload s4m > $O/plain_s4m.txt 2>&1 || exit 1
for w in s4m c2; do
  IBMGPU_EAGER=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/launches_$w.csv python tools/profile_step.py --workload $w > $O/ncu_launch_$w.log 2>&1
  IBMGPU_EAGER=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none -s 400 -c 150 --csv --log-file $O/traffic_$w.csv python tools/profile_step.py --workload $w \
      > $O/ncu_traffic_$w.log 2>&1
done
IBMGPU_EAGER=1 ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:"k_spmv_|k_xfer_|k_symv" -s 60 -c 16 -o $O/full_s4m python tools/profile_step.py --workload s4m > $O/ncu_full.log 2>&1
echo done > $O/done
