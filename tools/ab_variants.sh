# A/B of library builds in abtest/lib_<name>.so (make EXTRA=-D... OBJDIR=build/obj_ab, then copy):
#   gpurun -- bash tools/ab_variants.sh base v1 v2   -> gpurun_out/abv.log
mkdir -p gpurun_out
for rep in 1 2; do for v in "$@"; do IBMGPU_LIB=$PWD/abtest/lib_$v.so TAG=$v python tools/ab_iter.py s4m c2; done; done > gpurun_out/abv.log 2>&1
