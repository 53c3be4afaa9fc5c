# k1_grid: run-to-run variance and the cost of the pacing code on C4 / C5; K = 128 parity.
mkdir -p gpurun_out
timeout 1500 python tools/kernel_sweep.py --configs c4c,c4h,c5 --variants default,nopace,default,nopace > gpurun_out/r2u_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_sweep.log
timeout 900 python -m pytest tests/test_gpu_grid.py -q -m gpu -p no:cacheprovider -k "128" > gpurun_out/r2u_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_tests.log
