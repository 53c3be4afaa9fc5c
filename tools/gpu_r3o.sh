mkdir -p gpurun_out
timeout 900 python tools/kernel_sweep.py --configs c5,c4c --variants default,skip3,default,skip3 > gpurun_out/r3o_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r3o_sweep.log
