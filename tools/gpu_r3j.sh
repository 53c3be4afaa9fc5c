mkdir -p gpurun_out
(timeout 600 python tools/var3d_probe.py 128 32 8; timeout 600 python tools/var3d_probe.py 160 64 16; timeout 600 python tools/var3d_probe.py 128 16 4) > gpurun_out/r3j_var3d.log 2>&1; echo "rc=$?" >> gpurun_out/r3j_var3d.log
