# Fixes + final measurements: the CLI timing test, C3 full fixtures, then the measurement script.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cli.py "tests/test_gpu_full.py::test_full_fixtures_present" "tests/test_gpu_full.py::test_full_fast_parity_bars[c3_full_global4]" "tests/test_gpu_full.py::test_full_fast_parity_bars[c3_full_parallel]" -q -m gpu -p no:cacheprovider > gpurun_out/r3c_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3c_tests.log
bash tools/gpu_r2v.sh
