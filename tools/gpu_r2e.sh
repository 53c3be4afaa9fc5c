# Round-2 re-entry check: new-path parity (k1_stage, psolver, k=128, C5 128^3), sweep stage on/off, C5 bench + reference arm.
mkdir -p gpurun_out
nproc > gpurun_out/r2e_host.txt; free -g >> gpurun_out/r2e_host.txt
timeout 1500 python -m pytest tests/test_gpu_line.py tests/test_gpu_psolver.py tests/test_gpu_k128.py tests/test_gpu_fused.py "tests/test_gpu_full.py::test_full_fast_parity_bars[c5_full_128]" "tests/test_gpu_full.py::test_full_exact_bit_identical[c5_full_128]" -q -m gpu -p no:cacheprovider > gpurun_out/r2e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2e_smoke.log
timeout 1500 python tools/kernel_sweep.py --configs c5,c2,c4c,c4h,c3p,c1 --variants default --envs "BKG_K1_STAGE=0;BKG_K1_STAGE=1;BKG_K1_STAGE=1,BKG_STAGE_CTAS=2;BKG_K1_STAGE=1,BKG_STAGE_NS=3" > gpurun_out/r2e_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_sweep.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2e_bench_c5.json 2> gpurun_out/r2e_bench_c5.err; echo "rc=$?" >> gpurun_out/r2e_bench_c5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2e_ref_c5.json 2> gpurun_out/r2e_ref_c5.err; echo "rc=$?" >> gpurun_out/r2e_ref_c5.err
