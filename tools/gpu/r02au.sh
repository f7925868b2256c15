# round 2au: experiment: cold arena mapped as a head handle before the copies + the tail on a thread beside them (CRAC_COLD_HEAD_MIB)
mkdir -p gpurun_out/r02au
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -m gpu > gpurun_out/r02au/scale_tests.log 2>&1; tail -2 gpurun_out/r02au/scale_tests.log
CRAC_TRACE=1 timeout 600 python bench.py --steps 1 --warmup 1 --no-stall --no-cpu-baseline --no-incremental --no-verify > gpurun_out/r02au/trace.json 2> gpurun_out/r02au/trace.err
for rep in 1 2; do
for mb in 8192 0 4096; do
CRAC_COLD_HEAD_MIB=$mb timeout 900 python bench.py --steps 3 --warmup 2 --no-stall --no-cpu-baseline --no-incremental --no-verify > gpurun_out/r02au/c4_${mb}_$rep.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02au/c4_${mb}_$rep.json').read().splitlines()[-1]); print('c4 head=$mb', d['value'], d['e2e']['value'], d['per_gpu']['restart_ms'], d['per_gpu']['warm_restart']['restart_ms'], d['roofline']['frac'])"
done
done
