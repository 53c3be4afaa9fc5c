# k1_line at run length 64: parity tests and the C5 bench line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_line.py tests/test_gpu_fused.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r10_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r10_tests.log
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/r10_bench_c5.log 2>&1
