# round 2ax: does the nvidia-smi clock sampler's start-up stall the timed steps? sampler started at the timed region vs before the warm-up vs none
mkdir -p gpurun_out/r02ax
for rep in 1 2; do
for mode in timed warmup none; do
if [ $mode = none ]; then export CRAC_NO_CLOCKS=1; else unset CRAC_NO_CLOCKS; fi
CRAC_CLOCKS_AT=$mode timeout 900 python bench.py --steps 3 --warmup 3 --no-stall --no-cpu-baseline --no-incremental --no-verify > gpurun_out/r02ax/c4_${mode}_$rep.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02ax/c4_${mode}_$rep.json').read().splitlines()[-1]); print('c4 $mode', d['value'], d['e2e']['value'], d['per_gpu']['restart_ms'], d['per_gpu']['checkpoint_ms'], d['e2e']['teardown_ms_per_step'], (d.get('clocks') or {}).get('samples'))"
CRAC_CLOCKS_AT=$mode timeout 600 python bench.py --workload c2 --steps 8 --warmup 3 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02ax/c2_${mode}_$rep.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02ax/c2_${mode}_$rep.json').read().splitlines()[-1]); print('c2 $mode', d['value'], d['e2e']['value'], d['per_gpu']['restart_ms'], d['e2e']['teardown_ms_per_step'], d['roofline']['h2d_GBps_per_step'])"
done
done
