# round 2aj: C2 teardown outliers: async live-table destruction on / off
mkdir -p gpurun_out/r02aj
for rep in 1 2 3; do timeout 600 python bench.py --workload c2 --steps 8 --warmup 3 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02aj/c2_$rep.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02aj/c2_$rep.json').read().splitlines()[-1]); print('c2', d['value'], d['e2e']['value'], d['per_gpu']['restart_ms'], d['e2e']['teardown_ms_per_step'])"; done
nvidia-smi --query-gpu=name,memory.used,memory.total,clocks.sm --format=csv
free -g | head -2
