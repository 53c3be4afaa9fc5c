# K2/K3 L2 bulk prefetch distance sweep; C1 latency breakdown.
mkdir -p gpurun_out
timeout 1500 python tools/kernel_sweep.py --configs c5,c2,c4c,c3p --variants default,mpf1,mpf2,mpf4 > gpurun_out/r2w_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2w_sweep.log
timeout 300 python tools/c1_latency.py c1 > gpurun_out/r2w_c1.log 2>&1; echo "rc=$?" >> gpurun_out/r2w_c1.log
