# Round-2 measurements with k1_grid default: sweep, C5 bench + reference arm, secondary configs, launch list, ncu --set full (reports stay on the box; CSV pages come back).
mkdir -p gpurun_out
R=/tmp/ncu_r2v; mkdir -p $R
timeout 1500 python tools/kernel_sweep.py --configs c5,c2,c4c,c4h,c4g > gpurun_out/r2v_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2v_sweep.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2v_bench_c5.json 2> gpurun_out/r2v_bench_c5.err; echo "rc=$?" >> gpurun_out/r2v_bench_c5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2v_ref_c5.json 2> gpurun_out/r2v_ref_c5.err; echo "rc=$?" >> gpurun_out/r2v_ref_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2v_launches_c5.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/r2v_launches.log 2>&1; echo "rc=$?" >> gpurun_out/r2v_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_grid|k2_mma|k3_mma" -c 6 -o $R/c5 python tools/profile_run.py c5 2 > gpurun_out/r2v_c5_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/r2v_c5_ncu.log
timeout 600 ncu --set full --clock-control none -k regex:"k1_grid" -c 1 -o $R/c4 python tools/profile_run.py c4c 2 > gpurun_out/r2v_c4_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/r2v_c4_ncu.log
timeout 600 ncu --set full --clock-control none -k regex:"k1_grid|k2_mma|k3_mma" -c 6 -o $R/c2 python tools/profile_run.py c2 2 > gpurun_out/r2v_c2_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/r2v_c2_ncu.log
for c in c5 c4 c2; do ncu -i $R/$c.ncu-rep --page raw --csv > gpurun_out/r2v_ncu_$c.raw.csv 2>/dev/null; ncu -i $R/$c.ncu-rep --page details --csv > gpurun_out/r2v_ncu_$c.details.csv 2>/dev/null; done
ls -la $R > gpurun_out/r2v_ncu_ls.txt
for c in c2 c4c c4h c3p c1; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/r2v_bench_$c.json 2> gpurun_out/r2v_bench_$c.err; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2v_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2v_smoke.log
du -sh gpurun_out >> gpurun_out/r2v_ncu_ls.txt
