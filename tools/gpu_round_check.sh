# Round-end B200 check: full GPU suite, C2 bench line, C5 bench line (k1_line picked by the solver).
mkdir -p gpurun_out
timeout 2100 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r3_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r3_pytest_gpu.log
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/r3_bench_c2.log 2>&1
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/r3_bench_c5.log 2>&1
