# Round-2: k1_stage correctness (first K1 step vs oracle on all shapes, solves) and timing.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_line.py tests/test_gpu_psolver.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r2b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_tests.log
timeout 900 python tools/kernel_sweep.py --configs c5,c2,c4c,c4h,c3p,c3g,c1 --envs "BKG_K1_STAGE=0;BKG_K1_STAGE=1;BKG_K1_STAGE=1,BKG_STAGE_NS=3;BKG_K1_STAGE=1,BKG_STAGE_CTAS=2" > gpurun_out/r2b_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_sweep.log
