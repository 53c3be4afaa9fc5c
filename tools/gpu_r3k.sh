# VAR default (2-D and 3-D), final residual through K1: tests + C5/C2/C3 bench lines.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_grid.py tests/test_gpu_solver.py tests/test_gpu_irregular.py "tests/test_gpu_full.py::test_full_fast_parity_bars" tests/test_gpu_deferred.py tests/test_gpu_cli.py -q -m gpu -p no:cacheprovider > gpurun_out/r3k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3k_tests.log
for c in c5 c2 c3p c4c; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/r3k_bench_$c.json 2> gpurun_out/r3k_bench_$c.err; done
