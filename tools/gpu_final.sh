# Final check at HEAD: full GPU suite, then the measurement script.
bash tools/gpu_suite.sh
bash tools/gpu_r2v.sh
timeout 600 python bench.py --config c3g --steps 5 --warmup 3 --no-cpu > gpurun_out/r2v_bench_c3g.json 2> gpurun_out/r2v_bench_c3g.err
R=/tmp/ncu_final; mkdir -p $R
timeout 600 ncu --set full --clock-control none -k regex:"k1_grid2" -c 1 -o $R/c3 python tools/profile_run.py c3p 2 > gpurun_out/r2v_c3_ncu.log 2>&1
ncu -i $R/c3.ncu-rep --page raw --csv > gpurun_out/r2v_ncu_c3.raw.csv 2>/dev/null; ncu -i $R/c3.ncu-rep --page details --csv > gpurun_out/r2v_ncu_c3.details.csv 2>/dev/null
