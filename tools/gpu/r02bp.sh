# round 2bp: refill skips the ring copy of windows no scatter reads (CRAC_RING_SKIP, default on): GPU suite, then C4 and
# C2 with it on / off, alternating
mkdir -p gpurun_out/r02bp
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r02bp/gputests.log 2>&1; tail -3 gpurun_out/r02bp/gputests.log
for rep in 1 2; do
for m in 1 0; do
CRAC_RING_SKIP=$m timeout 900 python bench.py --steps 3 --warmup 3 --no-stall --no-cpu-baseline --no-incremental > gpurun_out/r02bp/c4_skip${m}_$rep.json 2>gpurun_out/r02bp/c4_skip${m}_$rep.err
python -c "
import json; d=json.loads(open('gpurun_out/r02bp/c4_skip${m}_$rep.json').read().splitlines()[-1]); r=d['roofline']
print('c4 skip=$m', d['value'], d['e2e']['value'], d['per_gpu']['checkpoint_ms'], d['per_gpu']['restart_ms'], r['h2d_GBps_per_step'], r['h2d_peak_GBps'], 'verified', d['verified']['ok'], d['e2e']['h2d_bytes_per_step'])"
done
done
for m in 1 0; do
CRAC_RING_SKIP=$m timeout 600 python bench.py --workload c2 --no-stall --no-cpu-baseline > gpurun_out/r02bp/c2_skip$m.json 2>gpurun_out/r02bp/c2_skip$m.err
python -c "
import json; d=json.loads(open('gpurun_out/r02bp/c2_skip$m.json').read().splitlines()[-1])
print('c2 skip=$m', d['value'], d['e2e']['value'], d['per_gpu']['restart_ms'], 'verified', d['verified']['ok'])"
done
