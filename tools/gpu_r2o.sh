# k1_grid: remaining parity tests, ring depth / z-chunk sweep, ncu --set full on C5 and C4.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_grid.py -q -m gpu -p no:cacheprovider > gpurun_out/r2o_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_tests.log
timeout 1500 python tools/kernel_sweep.py --configs c5,c4c,c2 --variants default --envs "BKG_K1_GRID=1,BKG_GRID_NS=2;BKG_K1_GRID=1,BKG_GRID_NS=3,BKG_GRID_ZCHUNK=16;BKG_K1_GRID=1,BKG_GRID_NS=3,BKG_GRID_ZCHUNK=32;BKG_K1_GRID=1,BKG_GRID_NS=3,BKG_GRID_ZCHUNK=128;BKG_K1_GRID=1,BKG_GRID_NS=3,BKG_GRID_ZCHUNK=256" > gpurun_out/r2o_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_sweep.log
export BKG_K1_GRID=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_grid" -c 1 -o gpurun_out/r2o_grid_c5 python tools/profile_run.py c5 2 > gpurun_out/r2o_ncu_c5.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_ncu_c5.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_grid" -c 1 -o gpurun_out/r2o_grid_c4 python tools/profile_run.py c4c 2 > gpurun_out/r2o_ncu_c4.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_ncu_c4.log
BKG_GRID_NS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_grid" -c 1 -o gpurun_out/r2o_grid_c5_ns3 python tools/profile_run.py c5 2 > gpurun_out/r2o_ncu_c5_ns3.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_ncu_c5_ns3.log
