# round 2bv: host-run pages (and pinned payloads) hashed and streamed into the image in one read with non-temporal
# stores (CRAC_HOST_NT, default on) against CRC then memcpy (=0): parity tests, then C3 alternating
mkdir -p gpurun_out/r02bv
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "c3 or managed or pinned or random" > gpurun_out/r02bv/tests.log 2>&1; tail -2 gpurun_out/r02bv/tests.log
for rep in 1 2 3; do
for m in 1 0; do
CRAC_HOST_NT=$m timeout 600 python bench.py --workload c3 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02bv/c3_nt${m}_$rep.json 2>gpurun_out/r02bv/c3_nt${m}_$rep.err
python -c "
import json; d=json.loads(open('gpurun_out/r02bv/c3_nt${m}_$rep.json').read().splitlines()[-1]); r=d['roofline']
print('c3 nt=$m', d['value'], d['e2e']['value'], d['per_gpu']['checkpoint_ms'], d['per_gpu']['restart_ms'], r['d2h_GBps_per_step'])"
done
done
