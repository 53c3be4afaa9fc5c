# resident kernel phase profile on C1; stage first-step tests at 16 warps.
mkdir -p gpurun_out
BKG_RESIDENT_PROF=1 timeout 300 python bench.py --config c1 --steps 2 --warmup 1 --no-cpu > gpurun_out/r2l_c1_prof.json 2> gpurun_out/r2l_c1_prof.err; echo "rc=$?" >> gpurun_out/r2l_c1_prof.err
timeout 900 python -m pytest tests/test_gpu_resident.py -q -m gpu -p no:cacheprovider > gpurun_out/r2l_resident.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_resident.log
timeout 1200 python -m pytest tests/test_gpu_line.py tests/test_gpu_psolver.py -q -m gpu -p no:cacheprovider > gpurun_out/r2l_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_tests.log
