# One-off B200 check of the k1_line variant: forced-line parity tests, K1 sweep over run lengths, ncu of both K1s on C2.
mkdir -p gpurun_out
BKG_K1_LINE=1 timeout 900 python -m pytest tests/test_gpu_line.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r2_tests_line.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2_tests_line.log
BKG_K1_LINE=1 timeout 900 python tools/kernel_sweep.py --configs c2,c3p,c5,c4c --variants lr4,lr8,lr16,default > gpurun_out/r2_sweep_line.log 2>&1
BKG_K1_LINE=0 timeout 600 python tools/kernel_sweep.py --configs c2,c3p,c5,c4c > gpurun_out/r2_sweep_wide.log 2>&1
for L in 0 1; do BKG_K1_LINE=$L timeout 600 ncu --set full --clock-control none -k regex:"k1_wide|k1_line" -c 1 -o gpurun_out/r2_k1_line$L python tools/profile_run.py c2 2 > gpurun_out/r2_ncu$L.log 2>&1; done
