# k1_grid2 (2-D y-march): parity + sweep on 2-D constant and C3 (variable, opt-in).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_grid.py -q -x -m gpu -p no:cacheprovider > gpurun_out/r3d_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3d_tests.log
timeout 1500 python tools/kernel_sweep.py --configs 0:1024:1024:1:64:16:hybrid,0:1024:1024:1:16:4:hybrid,c3p,c3g --variants default --envs "BKG_GRID_VAR=1;BKG_GRID_VAR=1,BKG_GRID2=0;BKG_K1_GRID=0;BKG_GRID_VAR=1,BKG_GRID_NS=3;BKG_GRID_VAR=1,BKG_GRID_NS=6;BKG_GRID_VAR=1,BKG_GRID_ZCHUNK=32;BKG_GRID_VAR=1,BKG_GRID_ZCHUNK=128" > gpurun_out/r3d_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r3d_sweep.log
