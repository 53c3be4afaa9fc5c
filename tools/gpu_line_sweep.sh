# k1_line run length / chunk sweep on C5 (BKG_K1_LINE=1), variants from tools/build_variants.sh.
mkdir -p gpurun_out
BKG_K1_LINE=1 timeout 900 python tools/kernel_sweep.py --configs c5 --variants lr128,lr256,lr64,default > gpurun_out/r9_sweep.log 2>&1
