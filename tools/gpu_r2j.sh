# 16-warp k1_stage + predicate-free slot loop: correctness, sweep, decomposition; resident kernel on C1.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_line.py tests/test_gpu_psolver.py tests/test_gpu_solver.py tests/test_gpu_kernels.py -q -m gpu -p no:cacheprovider > gpurun_out/r2j_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_tests.log
timeout 1500 python tools/kernel_sweep.py --configs c5,c2,c4c,c3p --variants default,nt2 --envs "BKG_K1_STAGE=1;BKG_K1_STAGE=1,BKG_STAGE_MINNS=2" > gpurun_out/r2j_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_sweep.log
timeout 900 python tools/kernel_sweep.py --configs c5,c2 --variants default --envs "BKG_K1_STAGE=1,BKG_STAGE_MINNS=2,BKG_STAGE_DEBUG=1;BKG_K1_STAGE=1,BKG_STAGE_MINNS=2,BKG_STAGE_DEBUG=2;BKG_K1_STAGE=1,BKG_STAGE_MINNS=2,BKG_STAGE_DEBUG=3" > gpurun_out/r2j_debug.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_debug.log
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/r2j_bench_c1.json 2> gpurun_out/r2j_bench_c1.err; echo "rc=$?" >> gpurun_out/r2j_bench_c1.err
BKG_RESIDENT=0 timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/r2j_bench_c1_off.json 2> gpurun_out/r2j_bench_c1_off.err; echo "rc=$?" >> gpurun_out/r2j_bench_c1_off.err
timeout 900 python -m pytest tests/test_gpu_full.py -q -m gpu -p no:cacheprovider -k "c1 or classical or hybrid4 or global4 or present" > gpurun_out/r2j_tests_full.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_tests_full.log
