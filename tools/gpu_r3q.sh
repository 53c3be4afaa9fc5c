# Isotropic 27-point path of k1_grid: parity (all 27-point cases) + sweep on / off.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_grid.py "tests/test_gpu_full.py::test_full_fast_parity_bars" tests/test_gpu_psolver.py -q -m gpu -p no:cacheprovider > gpurun_out/r3q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3q_tests.log
timeout 900 python tools/kernel_sweep.py --configs c4c,c4h,c4g --variants default --envs "BKG_GRID_ISO=1;BKG_GRID_ISO=0;BKG_GRID_ISO=1;BKG_GRID_ISO=0" > gpurun_out/r3q_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r3q_sweep.log
