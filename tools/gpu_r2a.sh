# Round-2 check: partitioned (generated) + full-size C5 parity, smoke, C5 bench, reference arm.
mkdir -p gpurun_out
nproc > gpurun_out/r2a_host.txt; free -g >> gpurun_out/r2a_host.txt; lscpu | head -20 >> gpurun_out/r2a_host.txt
timeout 900 python -m pytest tests/test_gpu_psolver.py tests/test_gpu_generate.py "tests/test_gpu_full.py::test_full_fast_parity_bars[c5_full_128]" "tests/test_gpu_full.py::test_full_exact_bit_identical[c5_full_128]" -q -m gpu -p no:cacheprovider > gpurun_out/r2a_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2a_smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2a_bench_c5.json 2> gpurun_out/r2a_bench_c5.err; echo "rc=$?" >> gpurun_out/r2a_bench_c5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2a_ref_c5.json 2> gpurun_out/r2a_ref_c5.err; echo "rc=$?" >> gpurun_out/r2a_ref_c5.err
