#!/bin/bash
# The checked build (device bounds checks, make CHECKED=1) under the GPU test suite: the stand-in
# for compute-sanitizer, which is closed on this GPU pool. Restores the normal build afterwards.
set -u
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
rm -f paper_1109_3524_b200/libibmgpu.so
make -j16 CHECKED=1 paper_1109_3524_b200/libibmgpu.so > "$OUT/checked_build.log" 2>&1 || { echo "checked build failed"; exit 1; }
nm -C paper_1109_3524_b200/libibmgpu.so > /dev/null; cuobjdump -sass paper_1109_3524_b200/libibmgpu.so | grep -c BPT.TRAP >> "$OUT/checked_build.log"
timeout 1500 python -m pytest tests -q -m gpu -k "not s4m_three" -p no:cacheprovider > "$OUT/checked_tests.log" 2>&1
echo "rc=$?" >> "$OUT/checked_tests.log"
python -c "import __graft_entry__ as g; g.smoke()" >> "$OUT/checked_tests.log" 2>&1
rm -f paper_1109_3524_b200/libibmgpu.so
make -j16 paper_1109_3524_b200/libibmgpu.so > /dev/null 2>&1
