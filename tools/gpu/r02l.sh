# round 2l: C2 cold restart A/B: single-run vs per-run premap, with and without tracing
mkdir -p gpurun_out/r02l
for rep in 1 2; do
for single in 1 0; do
  CRAC_PREMAP_SINGLE=$single timeout 600 python bench.py --workload c2 --steps 5 --warmup 3 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02l/c2_s${single}_$rep.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/r02l/c2_s${single}_$rep.json').read().splitlines()[-1]); print('single=$single rep=$rep', d['value'], d['e2e']['value'], d['per_gpu']['checkpoint_ms'], d['per_gpu']['restart_ms'], d['per_gpu']['warm_restart']['restart_ms'])"
done
done
CRAC_TRACE=1 timeout 600 python bench.py --workload c2 --steps 5 --warmup 3 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02l/c2_trace.json 2> gpurun_out/r02l/c2_trace.err
python -c "import json; d=json.loads(open('gpurun_out/r02l/c2_trace.json').read().splitlines()[-1]); print('trace', d['value'], d['per_gpu']['restart_ms'])"
