# K2/K3 TMA kernels: parity (solver-level tests with BKG_TMA23=1), sweep on/off; C1 clock check.
mkdir -p gpurun_out
export BKG_TMA23=1
timeout 1200 python -m pytest tests/test_gpu_grid.py tests/test_gpu_deferred.py tests/test_gpu_fused.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r2y_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2y_tests.log
unset BKG_TMA23
timeout 1500 python tools/kernel_sweep.py --configs c5,c2,c4c,c4h,c3p --variants default --envs "BKG_TMA23=0;BKG_TMA23=1" > gpurun_out/r2y_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2y_sweep.log
timeout 300 python tools/c1_latency.py c1 > gpurun_out/r2y_c1.log 2>&1; echo "rc=$?" >> gpurun_out/r2y_c1.log
