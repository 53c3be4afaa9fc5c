# Driver-like end-of-round check at HEAD: smoke(), default bench line, reference arm, launch list of the bench.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r7_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r7_smoke.log
timeout 400 python bench.py > gpurun_out/r7_bench.log 2>&1
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r7_bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r7_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/r7_ncu.log 2>&1
