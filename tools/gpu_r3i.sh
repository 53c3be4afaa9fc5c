# fast_bsolve (one-warp block solves) in every fused kernel: sweep, then the full suite.
mkdir -p gpurun_out
timeout 1500 python tools/kernel_sweep.py --configs c5,c2,c4c,c4h,c3p,c3g,c1,0:1024:1024:1:64:16:hybrid --variants default --envs "BKG_RESIDENT=0" > gpurun_out/r3i_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r3i_sweep.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r3i_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r3i_pytest_gpu.log
