# k1_grid 2x2 window version: parity, full-size fast parity (auto k1_grid), NS sweep.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_grid.py -q -m gpu -p no:cacheprovider > gpurun_out/r2p_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2p_tests.log
timeout 1500 python tools/kernel_sweep.py --configs c5,c4c,c4h,c2 --variants default --envs "BKG_GRID_NS=3;BKG_GRID_NS=4;BKG_GRID_NS=5" > gpurun_out/r2p_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2p_sweep.log
timeout 1800 python -m pytest tests/test_gpu_full.py tests/test_gpu_line.py -q -m gpu -p no:cacheprovider -k "fast_parity or large_system or parity_bars" > gpurun_out/r2p_full.log 2>&1; echo "rc=$?" >> gpurun_out/r2p_full.log
