# round 2bq: C2 with the ring skip on / off, 3 alternating rounds (r02bp's single C2 pair had one slow run)
mkdir -p gpurun_out/r02bq
for rep in 1 2 3; do
for m in 1 0; do
CRAC_RING_SKIP=$m timeout 600 python bench.py --workload c2 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02bq/c2_skip${m}_$rep.json 2>gpurun_out/r02bq/c2_skip${m}_$rep.err
python -c "
import json; d=json.loads(open('gpurun_out/r02bq/c2_skip${m}_$rep.json').read().splitlines()[-1]); r=d['roofline']
print('c2 skip=$m', d['value'], d['e2e']['value'], d['per_gpu']['checkpoint_ms'], d['per_gpu']['restart_ms'], r['h2d_GBps_per_step'], d['e2e']['h2d_bytes_per_step'])"
done
done
