mkdir -p gpurun_out
for rep in 1 2; do for v in base w3 a6 s5; do IBMGPU_LIB=$PWD/abtest/lib_$v.so TAG=$v python tools/ab_iter.py s4m c2; done; done > gpurun_out/abv.log 2>&1
