# No sliced-ELL copy when K1 is a grid kernel: parity subset + bench lines.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_grid.py tests/test_gpu_solver.py "tests/test_gpu_full.py::test_full_fast_parity_bars" tests/test_gpu_psolver.py tests/test_gpu_line.py tests/test_gpu_cli.py tests/test_gpu_cpp.py tests/test_gpu_deferred.py -q -m gpu -p no:cacheprovider > gpurun_out/r3m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3m_tests.log
for c in c5 c2; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/r3m_bench_$c.json 2> gpurun_out/r3m_bench_$c.err; done
