# k1_stage with the segment list prefetched by every warp: correctness + sweep.
mkdir -p gpurun_out
BKG_K1_STAGE=1 timeout 600 python -m pytest tests/test_gpu_line.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r2g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_tests.log
timeout 900 python tools/kernel_sweep.py --configs c5,c2,c4c,c3p --variants default --envs "BKG_K1_STAGE=1;BKG_K1_STAGE=1,BKG_STAGE_CTAS=2" > gpurun_out/r2g_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_sweep.log
