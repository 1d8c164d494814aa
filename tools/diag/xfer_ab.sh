# A/B of the level-0 transfer tile grid (IBMGPU_XFER_CTAS: 0 = one CTA per tile) on S-4M and C2
O=gpurun_out/xprof; mkdir -p $O
python tools/diag/xfer_probe.py c2 s4m > $O/probe.log 2>&1
for i in 1 2; do IBMGPU_XFER_CTAS=0 TAG=pertile python tools/ab_iter.py s4m c2; TAG=persist python tools/ab_iter.py s4m c2; IBMGPU_XFER_CTAS=2 TAG=persist2 python tools/ab_iter.py s4m c2; done > $O/ab.log 2>&1
[ -n "$NO_NCU" ] || IBMGPU_EAGER=1 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_xfer" -s 6 -c 3 -o $O/xfer3_s4m python tools/profile_step.py --workload s4m > $O/ncu.log 2>&1
