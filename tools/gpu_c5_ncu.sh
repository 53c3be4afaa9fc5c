# ncu --set full of the C5 fused iteration (K1 as the solver picks it, K2, both K3 modes) and of k1_wide in row order.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_line|k1_wide|k2_mma|k3_mma|k2_update|k3_update" -c 4 -o gpurun_out/r4_c5 python tools/profile_run.py c5 2 > gpurun_out/r4_c5_ncu.log 2>&1
BKG_K1_LINE=0 BKG_K1_ZB=0 timeout 900 ncu --set full --clock-control none -k regex:"k1_wide" -c 1 -o gpurun_out/r5_c5_wide python tools/profile_run.py c5 2 > gpurun_out/r5_c5_ncu.log 2>&1
