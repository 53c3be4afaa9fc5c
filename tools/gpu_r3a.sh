# k1_grid: planes outside the tensor skipped + tail emit, 2-D grids; parity + sweep.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_grid.py tests/test_gpu_psolver.py -q -x -m gpu -p no:cacheprovider > gpurun_out/r3a_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3a_tests.log
timeout 1500 python tools/kernel_sweep.py --configs c5,c2,c4c,0:1024:1024:1:64:16:hybrid,0:1024:1024:1:16:4:hybrid --variants default --envs "BKG_K1_GRID=1;BKG_K1_GRID=0" > gpurun_out/r3a_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r3a_sweep.log
