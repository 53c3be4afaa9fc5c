mkdir -p gpurun_out
for v in a b; do timeout 600 python bench.py --config c3p --steps 3 --warmup 2 --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3p default', d['value'], d['e2e']['value'])"; done > gpurun_out/r3l_c3p.log 2>&1
BKG_GRID_VAR=0 timeout 600 python bench.py --config c3p --steps 3 --warmup 2 --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3p VAR=0', d['value'], d['e2e']['value'])" >> gpurun_out/r3l_c3p.log 2>&1
timeout 600 python tools/e2e_breakdown.py c3p >> gpurun_out/r3l_c3p.log 2>&1
