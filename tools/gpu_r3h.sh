# Resident kernel with warp_bsolve + parallel cta_reduce: tests, C1 latency.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_resident.py tests/test_gpu_solver.py -q -m gpu -p no:cacheprovider > gpurun_out/r3h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3h_tests.log
timeout 120 python tools/c1_clocks.py > gpurun_out/r3h_c1.log 2>&1; echo "rc=$?" >> gpurun_out/r3h_c1.log
timeout 300 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/r3h_bench_c1.json 2> gpurun_out/r3h_bench_c1.err
