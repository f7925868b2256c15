# round 2bt: early ring windows queued before a big cold arena's head map (CRAC_EARLY_FIRST, default on) against after
# it (=0): GPU parity + scale tests, then C4 alternating
mkdir -p gpurun_out/r02bt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q > gpurun_out/r02bt/tests.log 2>&1; tail -2 gpurun_out/r02bt/tests.log
for rep in 1 2 3; do
for m in 1 0; do
CRAC_EARLY_FIRST=$m timeout 900 python bench.py --steps 3 --warmup 3 --no-stall --no-cpu-baseline --no-incremental --no-verify > gpurun_out/r02bt/c4_early${m}_$rep.json 2>gpurun_out/r02bt/c4_early${m}_$rep.err
python -c "
import json; d=json.loads(open('gpurun_out/r02bt/c4_early${m}_$rep.json').read().splitlines()[-1]); r=d['roofline']
print('c4 early_first=$m', d['value'], d['e2e']['value'], d['per_gpu']['checkpoint_ms'], d['per_gpu']['restart_ms'], r['h2d_GBps_per_step'], r['frac'])"
done
done
