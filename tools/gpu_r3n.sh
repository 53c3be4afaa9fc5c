# ncu --set full of two whole C5 / C2 iterations (K3 skip and flush launches both).
mkdir -p gpurun_out
R=/tmp/ncu_r3n; mkdir -p $R
timeout 900 ncu --set full --clock-control none -k regex:"k1_grid|k2_mma|k3_mma" -c 6 -o $R/c5 python tools/profile_run.py c5 2 > gpurun_out/r3n_c5_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/r3n_c5_ncu.log
timeout 600 ncu --set full --clock-control none -k regex:"k1_grid|k2_mma|k3_mma" -c 6 -o $R/c2 python tools/profile_run.py c2 2 > gpurun_out/r3n_c2_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/r3n_c2_ncu.log
for c in c5 c2; do ncu -i $R/$c.ncu-rep --page raw --csv > gpurun_out/r3n_ncu_$c.raw.csv 2>/dev/null; ncu -i $R/$c.ncu-rep --page details --csv > gpurun_out/r3n_ncu_$c.details.csv 2>/dev/null; done
