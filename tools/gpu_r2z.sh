# Block-vector allocation skew sweep (power-of-two sized vectors alias in L2 / DRAM banks).
mkdir -p gpurun_out
timeout 2400 python tools/kernel_sweep.py --configs c5,c2,c3p,c4c --variants default --envs "BKG_VEC_SKEW=0;BKG_VEC_SKEW=256;BKG_VEC_SKEW=2304;BKG_VEC_SKEW=4352;BKG_VEC_SKEW=33024;BKG_VEC_SKEW=139520;BKG_VEC_SKEW=1048832;BKG_VEC_SKEW=4352,BKG_TMA23=1;BKG_VEC_SKEW=139520,BKG_TMA23=1" > gpurun_out/r2z_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2z_sweep.log
