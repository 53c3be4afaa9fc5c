# psolver with k1_grid parts; grid + line + psolver test files; default sweep on all configs.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_psolver.py tests/test_gpu_grid.py -q -m gpu -p no:cacheprovider > gpurun_out/r2t_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_tests.log
timeout 1500 python tools/kernel_sweep.py --configs c5,c2,c4c,c4h,c4g,c3p,c3g,c1 --variants default > gpurun_out/r2t_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_sweep.log
