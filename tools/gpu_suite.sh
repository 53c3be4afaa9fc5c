# Full GPU suite at HEAD.
mkdir -p gpurun_out
timeout 2100 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r11_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r11_pytest_gpu.log
