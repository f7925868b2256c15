# round 2y: replay on its own thread in the early refill; parity + C2 bench x3 (8 steps)
mkdir -p gpurun_out/r02y
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_engine_stress.py tests/test_gpu_interpose.py -x -q > gpurun_out/r02y/gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02y/gputests.log
for rep in 1 2 3; do
  timeout 600 python bench.py --workload c2 --steps 8 --warmup 3 --no-stall --no-cpu-baseline > gpurun_out/r02y/c2_$rep.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/r02y/c2_$rep.json').read().splitlines()[-1]); print('rep=$rep', d['value'], d['e2e']['value'], d['per_gpu']['checkpoint_ms'], d['per_gpu']['restart_ms'], d['per_gpu']['warm_restart']['restart_ms'], d['roofline']['frac'], d['verified']['ok'])"
done
CRAC_TRACE=1 timeout 600 python bench.py --workload c2 --steps 3 --warmup 2 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02y/c2_trace.json 2> gpurun_out/r02y/c2_trace.err
