# k1_stage without per-block CTA barriers: correctness + sweep (NS / CTAs per SM / TPW).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_line.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r2d_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_tests.log
timeout 1500 python tools/kernel_sweep.py --configs c5,c2,c4c,c3p,c1 --variants default,tpw2 --envs "BKG_K1_STAGE=0;BKG_K1_STAGE=1;BKG_K1_STAGE=1,BKG_STAGE_CTAS=2" > gpurun_out/r2d_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_sweep.log
