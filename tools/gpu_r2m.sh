# Round-2 baseline at HEAD: full GPU suite, smoke, C5 bench + reference arm, launch list, ncu --set full of the C5 iteration.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2m_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2m_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2m_smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2m_bench_c5.json 2> gpurun_out/r2m_bench_c5.err; echo "rc=$?" >> gpurun_out/r2m_bench_c5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2m_ref_c5.json 2> gpurun_out/r2m_ref_c5.err; echo "rc=$?" >> gpurun_out/r2m_ref_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2m_launches_c5.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/r2m_launches.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_line|k1_wide|k2_mma|k3_mma|k2_update|k3_update" -c 4 -o gpurun_out/r2m_c5 python tools/profile_run.py c5 2 > gpurun_out/r2m_c5_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_c5_ncu.log
