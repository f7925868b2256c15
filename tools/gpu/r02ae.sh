# round 2ae: where the e2e-only time goes (session close, arena release), C4 and C2
mkdir -p gpurun_out/r02ae
for rep in 1 2; do
timeout 900 python bench.py --steps 4 --warmup 2 --no-stall --no-cpu-baseline --no-incremental --no-verify > gpurun_out/r02ae/c4_$rep.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/r02ae/c4_$rep.json').read().splitlines()[-1]); print('c4', d['value'], d['e2e']['value'], d['e2e']['teardown_ms_per_step'])"
timeout 600 python bench.py --workload c2 --steps 8 --warmup 3 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02ae/c2_$rep.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02ae/c2_$rep.json').read().splitlines()[-1]); print('c2', d['value'], d['e2e']['value'], d['e2e']['teardown_ms_per_step'])"
done
