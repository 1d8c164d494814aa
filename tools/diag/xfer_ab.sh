# A/B of the level-0 stencil transfers (IBMGPU_XFER0) on S-4M and C2, + ncu of the xfer kernels
O=gpurun_out/xprof; mkdir -p $O
python tools/diag/xfer_probe.py c2 s4m > $O/probe.log 2>&1
for i in 1 2; do IBMGPU_XFER0=0 TAG=off python tools/ab_iter.py s4m c2; TAG=on python tools/ab_iter.py s4m c2; done > $O/ab.log 2>&1
[ -n "$NO_NCU" ] || IBMGPU_EAGER=1 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_xfer" -s 6 -c 3 -o $O/xfer2_s4m python tools/profile_step.py --workload s4m > $O/ncu.log 2>&1
