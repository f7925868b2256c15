# round 2ah: threaded cold map (default for arenas <= 16 GiB): parity suites + C2 x2
mkdir -p gpurun_out/r02ah
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r02ah/gputests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02ah/gputests.log
for rep in 1 2; do timeout 600 python bench.py --workload c2 --steps 8 --warmup 3 --no-stall --no-cpu-baseline > gpurun_out/r02ah/c2_$rep.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02ah/c2_$rep.json').read().splitlines()[-1]); print('c2', d['value'], d['e2e']['value'], d['per_gpu']['checkpoint_ms'], d['per_gpu']['restart_ms'], d['roofline']['frac'], d['verified']['ok'], d['e2e']['teardown_ms_per_step'])"; done
