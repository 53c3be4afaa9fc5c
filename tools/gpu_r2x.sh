mkdir -p gpurun_out
timeout 300 python tools/c1_latency.py c1 > gpurun_out/r2x_c1.log 2>&1; echo "rc=$?" >> gpurun_out/r2x_c1.log
