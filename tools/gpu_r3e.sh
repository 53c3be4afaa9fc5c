# 2-D variable coefficients default on: grid tests, full-size C3 fixtures, C3 bench lines, trimmed exact test.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_grid.py tests/test_gpu_line.py "tests/test_gpu_full.py::test_full_fast_parity_bars" "tests/test_gpu_full.py::test_full_exact_bit_identical[c4_full_global4]" tests/test_gpu_solver.py tests/test_gpu_irregular.py -q -m gpu -p no:cacheprovider --durations=5 > gpurun_out/r3e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3e_tests.log
for c in c3p c3g; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/r3e_bench_$c.json 2> gpurun_out/r3e_bench_$c.err; done
R=/tmp/ncu_r3e; mkdir -p $R
timeout 600 ncu --set full --clock-control none -k regex:"k1_grid2" -c 1 -o $R/c3 python tools/profile_run.py c3p 2 > gpurun_out/r3e_c3_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/r3e_c3_ncu.log
ncu -i $R/c3.ncu-rep --page raw --csv > gpurun_out/r3e_ncu_c3.raw.csv 2>/dev/null; ncu -i $R/c3.ncu-rep --page details --csv > gpurun_out/r3e_ncu_c3.details.csv 2>/dev/null
