# round 2af: is the clock sampler (nvidia-smi -lms 200) what stalls the arena release?
mkdir -p gpurun_out/r02af
for rep in 1 2; do
for nc in 1 0; do
if [ $nc = 1 ]; then export CRAC_NO_CLOCKS=1; else unset CRAC_NO_CLOCKS; fi
timeout 600 python bench.py --workload c2 --steps 8 --warmup 3 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02af/c2_${nc}_$rep.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02af/c2_${nc}_$rep.json').read().splitlines()[-1]); print('c2 noclocks=$nc', d['value'], d['e2e']['value'], d['e2e']['teardown_ms_per_step'])"
done
done
