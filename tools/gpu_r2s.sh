# k1_grid pacing sweep (fixed segment accounting).
mkdir -p gpurun_out
timeout 1500 python tools/kernel_sweep.py --configs c5,c2 --variants default --envs "BKG_GRID_SYNC=0;BKG_GRID_SYNC=2,BKG_GRID_LEAD=2;BKG_GRID_SYNC=2,BKG_GRID_LEAD=4;BKG_GRID_SYNC=4,BKG_GRID_LEAD=1;BKG_GRID_SYNC=4,BKG_GRID_LEAD=2;BKG_GRID_SYNC=8,BKG_GRID_LEAD=1;BKG_GRID_SYNC=8,BKG_GRID_LEAD=2;BKG_GRID_SYNC=16,BKG_GRID_LEAD=1" > gpurun_out/r2s_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_sweep.log
