# k1_grid with variable coefficients (DIA tiles): parity + C3 sweep.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_grid.py -q -x -m gpu -p no:cacheprovider > gpurun_out/r3b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3b_tests.log
timeout 1500 python tools/kernel_sweep.py --configs c3p,c3g,c5,c4c --variants default --envs "BKG_K1_GRID=1;BKG_K1_GRID=0" > gpurun_out/r3b_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r3b_sweep.log
