# k1_grid lockstep pacing sweep (segment length, lead), parity re-check.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grid.py -q -x -m gpu -p no:cacheprovider > gpurun_out/r2r_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_tests.log
timeout 1500 python tools/kernel_sweep.py --configs c5,c2 --variants default --envs "BKG_GRID_NS=3,BKG_GRID_SYNC=0;BKG_GRID_NS=3;BKG_GRID_NS=3,BKG_GRID_SYNC=1,BKG_GRID_LEAD=2;BKG_GRID_NS=3,BKG_GRID_SYNC=1,BKG_GRID_LEAD=1;BKG_GRID_NS=3,BKG_GRID_SYNC=4,BKG_GRID_LEAD=1;BKG_GRID_NS=3,BKG_GRID_SYNC=2,BKG_GRID_LEAD=1;BKG_GRID_NS=4,BKG_GRID_SYNC=2,BKG_GRID_LEAD=1;BKG_GRID_NS=5,BKG_GRID_SYNC=2,BKG_GRID_LEAD=1" > gpurun_out/r2r_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_sweep.log
BKG_GRID_NS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_grid" -c 1 -o gpurun_out/r2r_grid_c5 python tools/profile_run.py c5 2 > gpurun_out/r2r_ncu_c5.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_ncu_c5.log
