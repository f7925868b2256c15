# round 2ag: experiment: cold arena map on a thread beside the early windows + parse (CRAC_MAP_BESIDE)
mkdir -p gpurun_out/r02ag
for rep in 1 2; do
for mb in 1 0; do
CRAC_MAP_BESIDE=$mb timeout 600 python bench.py --workload c2 --steps 8 --warmup 3 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02ag/c2_${mb}_$rep.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02ag/c2_${mb}_$rep.json').read().splitlines()[-1]); print('c2 beside=$mb', d['value'], d['e2e']['value'], d['per_gpu']['restart_ms'], d['per_gpu']['warm_restart']['restart_ms'])"
CRAC_MAP_BESIDE=$mb timeout 900 python bench.py --steps 3 --warmup 2 --no-stall --no-cpu-baseline --no-incremental --no-verify > gpurun_out/r02ag/c4_${mb}_$rep.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02ag/c4_${mb}_$rep.json').read().splitlines()[-1]); print('c4 beside=$mb', d['value'], d['e2e']['value'], d['per_gpu']['restart_ms'])"
done
done
