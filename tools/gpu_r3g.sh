mkdir -p gpurun_out
R=/tmp/ncu_r3g; mkdir -p $R
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_resident" -c 1 -o $R/c1 python tools/c1_clocks.py > gpurun_out/r3g_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/r3g_ncu.log
ncu -i $R/c1.ncu-rep --page raw --csv > gpurun_out/r3g_ncu_c1.raw.csv 2>/dev/null
ncu -i $R/c1.ncu-rep --page details --csv > gpurun_out/r3g_ncu_c1.details.csv 2>/dev/null
ncu -i $R/c1.ncu-rep --page source --csv > gpurun_out/r3g_ncu_c1.source.csv 2>/dev/null
ls -la $R gpurun_out/r3g* > gpurun_out/r3g_ls.txt
