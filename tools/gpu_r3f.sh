mkdir -p gpurun_out
timeout 120 python tools/c1_clocks.py > gpurun_out/r3f_c1_clocks.log 2>&1; echo "rc=$?" >> gpurun_out/r3f_c1_clocks.log
