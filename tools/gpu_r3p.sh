# compute-sanitizer memcheck over the new kernels (k1_grid, k1_grid2 + DIA tiles, warp_bsolve, resident) on small cases.
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest "tests/test_gpu_grid.py::test_grid_first_step" "tests/test_gpu_grid.py::test_grid_variable_coefficients_and_rejects" "tests/test_gpu_grid.py::test_grid_first_step_z_chunks" tests/test_gpu_resident.py "tests/test_gpu_psolver.py::test_grid_parts" -q -x -m gpu -p no:cacheprovider -k "not 128" > gpurun_out/r3p_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r3p_memcheck.log
tail -c 3000 gpurun_out/r3p_memcheck.log > gpurun_out/r3p_memcheck_tail.log
