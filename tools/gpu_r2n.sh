# k1_grid first contact: parity tests, then the sweep against the CSR K1s.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_grid.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r2n_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_tests.log
timeout 1500 python tools/kernel_sweep.py --configs c5,c2,c4c,c4h --variants default --envs "BKG_K1_GRID=0;BKG_K1_GRID=1;BKG_K1_GRID=1,BKG_GRID_NS=4;BKG_K1_GRID=1,BKG_GRID_NS=3" > gpurun_out/r2n_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_sweep.log
