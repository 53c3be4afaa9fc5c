# k1_stage decomposition: TMA fill alone (debug 1), compute alone (debug 2), both; ncu on C2.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_psolver.py "tests/test_gpu_line.py::test_line_and_wide_agree_on_large_system" -q -m gpu -p no:cacheprovider > gpurun_out/r2i_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_tests.log
timeout 900 python tools/kernel_sweep.py --configs c5,c2 --variants default --envs "BKG_K1_STAGE=1,BKG_STAGE_MINNS=2;BKG_K1_STAGE=1,BKG_STAGE_MINNS=2,BKG_STAGE_DEBUG=1;BKG_K1_STAGE=1,BKG_STAGE_MINNS=2,BKG_STAGE_DEBUG=2;BKG_K1_STAGE=1,BKG_STAGE_MINNS=2,BKG_STAGE_DEBUG=3" > gpurun_out/r2i_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_sweep.log
export BKG_K1_STAGE=1 BKG_STAGE_MINNS=2
timeout 300 python tools/profile_run.py c2 3 > gpurun_out/r2i_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_stage -c 1 -o gpurun_out/r2i_stage_c2 python tools/profile_run.py c2 3 > gpurun_out/r2i_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r2i_ncu.log
