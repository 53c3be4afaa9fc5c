# L2 stride prefetch in k1_line / k1_wide: sweep; resident kernel tests.
mkdir -p gpurun_out
timeout 1500 python tools/kernel_sweep.py --configs c5,c2,c4c,c3p --variants pf0,default,pf1,pf4,wpf > gpurun_out/r2k_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_sweep.log
timeout 900 python -m pytest tests/test_gpu_resident.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r2k_resident.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_resident.log
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_kernels.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r2k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_tests.log
