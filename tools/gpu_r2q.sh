# k1_grid: 8x2 vs 16x1 row groups (window form both), ring depth; ncu of the 8x2 version on C5.
mkdir -p gpurun_out
timeout 1500 python tools/kernel_sweep.py --configs c5,c4c,c2 --variants default,arr0 --envs "BKG_GRID_NS=3;BKG_GRID_NS=2;BKG_GRID_NS=4" > gpurun_out/r2q_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_sweep.log
BKG_GRID_NS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_grid" -c 1 -o gpurun_out/r2q_grid_c5 python tools/profile_run.py c5 2 > gpurun_out/r2q_ncu_c5.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_ncu_c5.log
