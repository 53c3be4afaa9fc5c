# Box-blocked k1_stage: correctness (all K1 shapes, psolver split, k=128), box/ring sweeps, NT/U variants.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_line.py tests/test_gpu_psolver.py tests/test_gpu_k128.py -q -m gpu -p no:cacheprovider > gpurun_out/r2h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_tests.log
timeout 1500 python tools/kernel_sweep.py --configs c5,c2,c4c,c3p --variants default --envs "BKG_K1_STAGE=0;BKG_K1_STAGE=1;BKG_K1_STAGE=1,BKG_STAGE_MINNS=2;BKG_K1_STAGE=1,BKG_STAGE_BOX=0;BKG_K1_STAGE=1,BKG_STAGE_BOX=0,BKG_STAGE_TPW=4" > gpurun_out/r2h_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_sweep.log
timeout 900 python tools/kernel_sweep.py --configs c5,c2,c4c --variants nt1u8,nt1u4,nt2u8 --envs "BKG_K1_STAGE=1" > gpurun_out/r2h_variants.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_variants.log
