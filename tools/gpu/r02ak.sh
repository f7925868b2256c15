# round 2ak: C2 A/B beside map on/off, alternating, 3 pairs (teardown + restart variance)
mkdir -p gpurun_out/r02ak
for rep in 1 2 3; do for mb in 1 0; do
CRAC_MAP_BESIDE=$mb timeout 600 python bench.py --workload c2 --steps 8 --warmup 3 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02ak/c2_${mb}_$rep.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02ak/c2_${mb}_$rep.json').read().splitlines()[-1]); t=d['e2e']['teardown_ms_per_step']; print('c2 beside=$mb', d['value'], d['e2e']['value'], d['per_gpu']['restart_ms'], 'release max', max(b for a,b in t))"
done; done
