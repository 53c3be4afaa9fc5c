# k1_stage: correctness on all K1 shapes + one ncu --set full capture on C2.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_line.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r2c_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_tests.log
timeout 300 python tools/profile_run.py c2 3 > gpurun_out/r2c_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_stage -c 2 -o gpurun_out/r2c_stage_c2 python tools/profile_run.py c2 3 > gpurun_out/r2c_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r2c_ncu.log
