# Quick B200 check of the built library: smoke + the grid-kernel parity file + one bench line.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/quick_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/quick_smoke.log
timeout 900 python -m pytest tests/test_gpu_grid.py tests/test_gpu_resident.py -q -m gpu -p no:cacheprovider > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err; echo "rc=$?" >> gpurun_out/quick_bench.err
