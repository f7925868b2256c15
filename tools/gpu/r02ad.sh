# round 2ad: A/B exact-end direct runs (scatter-free windows) vs tile-aligned runs, C4 and C2 alternating
mkdir -p gpurun_out/r02ad
for rep in 1 2 3; do
for ex in 1 0; do
CRAC_EXACT_DIRECT=$ex timeout 900 python bench.py --steps 3 --warmup 2 --no-stall --no-cpu-baseline --no-incremental --no-verify > gpurun_out/r02ad/c4_${ex}_$rep.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/r02ad/c4_${ex}_$rep.json').read().splitlines()[-1]); r=d['roofline']; print('c4 exact=$ex', d['value'], d['e2e']['value'], d['per_gpu']['restart_ms'], r['h2d_GBps_per_step'], d['gpu_launches'])"
done
done
for rep in 1 2; do
for ex in 1 0; do
CRAC_EXACT_DIRECT=$ex timeout 600 python bench.py --workload c2 --steps 8 --warmup 3 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02ad/c2_${ex}_$rep.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02ad/c2_${ex}_$rep.json').read().splitlines()[-1]); print('c2 exact=$ex', d['value'], d['e2e']['value'], d['per_gpu']['restart_ms'])"
done
done
