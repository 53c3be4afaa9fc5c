# Re-run the r2e failures after the fixes; ncu --set full of k1_stage on C2; C5 bench with the register-gather K1.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_psolver.py tests/test_gpu_k128.py tests/test_gpu_fused.py -q -m gpu -p no:cacheprovider > gpurun_out/r2f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_tests.log
BKG_K1_STAGE=1 timeout 300 python tools/profile_run.py c2 3 > gpurun_out/r2f_plain.log 2>&1 && \
BKG_K1_STAGE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_stage -c 1 -o gpurun_out/r2f_stage_c2 python tools/profile_run.py c2 3 > gpurun_out/r2f_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r2f_ncu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2f_bench_c5.json 2> gpurun_out/r2f_bench_c5.err; echo "rc=$?" >> gpurun_out/r2f_bench_c5.err
