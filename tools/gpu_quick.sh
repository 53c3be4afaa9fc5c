# Quick B200 check: k1_line parity tests and smoke().
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_line.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r12_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r12_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r12_tests.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r12_tests.log
