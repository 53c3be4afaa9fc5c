# Full GPU suite at HEAD (+ the 40 slowest tests).
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=40 > gpurun_out/suite_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/suite_pytest_gpu.log
