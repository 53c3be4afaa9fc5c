# B200 check of the plane-blocked K1 order: parity tests, C5 K1 sweep (blocked k1_wide vs k1_line vs row order), ncu DRAM bytes.
# (the blocked-order tests, tests/test_gpu_zblock.py, went with the reverted code; see profiles/zblock_r01/)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_line.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r6_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r6_tests.log
for v in "BKG_K1_LINE=0 BKG_K1_ZB=1" "BKG_K1_LINE=0 BKG_K1_ZB=1 BKG_K1_ZB_ROWS=4096" "BKG_K1_LINE=0 BKG_K1_ZB=1 BKG_K1_ZB_ROWS=16384" "BKG_K1_LINE=1 BKG_K1_ZB=0" "BKG_K1_LINE=0 BKG_K1_ZB=0"; do echo "$v" >> gpurun_out/r6_sweep.log; env $v timeout 300 python tools/kernel_sweep.py --configs c5 >> gpurun_out/r6_sweep.log 2>&1; done
timeout 300 python tools/kernel_sweep.py --configs c2,c3p,c4c > gpurun_out/r6_sweep_others.log 2>&1
BKG_K1_LINE=0 BKG_K1_ZB=1 timeout 600 ncu --set full --clock-control none -k regex:"k1_wide" -c 1 -o gpurun_out/r6_c5_zb python tools/profile_run.py c5 2 > gpurun_out/r6_ncu.log 2>&1
