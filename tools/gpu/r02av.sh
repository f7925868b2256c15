# round 2av: split cold map (head handle + tail on a thread) with the old arena's release overlapping the refill (release_later) vs before it
mkdir -p gpurun_out/r02av
timeout 1200 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -x -q -m gpu -k "two_handle or cold_restart or regenerated or c1_full" > gpurun_out/r02av/tests.log 2>&1; tail -2 gpurun_out/r02av/tests.log
CRAC_TRACE=1 timeout 600 python bench.py --steps 2 --warmup 1 --no-stall --no-cpu-baseline --no-incremental --no-verify > gpurun_out/r02av/trace.json 2> gpurun_out/r02av/trace.err
for rep in 1 2; do
for cfg in "0 8192" "1 8192" "0 16384"; do
set -- $cfg
CRAC_SYNC_RELEASE=$1 CRAC_COLD_HEAD_MIB=$2 timeout 900 python bench.py --steps 3 --warmup 2 --no-stall --no-cpu-baseline --no-incremental --no-verify > gpurun_out/r02av/c4_$1_$2_$rep.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02av/c4_$1_$2_$rep.json').read().splitlines()[-1]); print('c4 sync=$1 head=$2', d['value'], d['e2e']['value'], d['per_gpu']['restart_ms'], d['roofline']['frac'], d['e2e']['teardown_ms_per_step'])"
done
CRAC_SYNC_RELEASE=0 timeout 600 python bench.py --workload c2 --steps 8 --warmup 3 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02av/c2_0_$rep.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02av/c2_0_$rep.json').read().splitlines()[-1]); print('c2 sync=0', d['value'], d['e2e']['value'], d['per_gpu']['restart_ms'], d['e2e']['teardown_ms_per_step'])"
CRAC_SYNC_RELEASE=1 timeout 600 python bench.py --workload c2 --steps 8 --warmup 3 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02av/c2_1_$rep.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02av/c2_1_$rep.json').read().splitlines()[-1]); print('c2 sync=1', d['value'], d['e2e']['value'], d['per_gpu']['restart_ms'], d['e2e']['teardown_ms_per_step'])"
done
