# round 2n: pinned payloads hashed on the host; cold refill maps a dense arena whole before the parse (A/B)
mkdir -p gpurun_out/r02n
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_kernels.py -x -q > gpurun_out/r02n/gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02n/gputests.log
for rep in 1 2; do
for fm in 1 0; do
  CRAC_COLD_FULLMAP=$fm timeout 600 python bench.py --workload c2 --steps 5 --warmup 3 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02n/c2_fm${fm}_$rep.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/r02n/c2_fm${fm}_$rep.json').read().splitlines()[-1]); print('fullmap=$fm rep=$rep', d['value'], d['e2e']['value'], d['per_gpu']['checkpoint_ms'], d['per_gpu']['restart_ms'], d['per_gpu']['warm_restart']['restart_ms'])"
done
done
timeout 900 python bench.py --steps 3 --warmup 2 --no-stall --no-cpu-baseline --no-incremental > gpurun_out/r02n/c4.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/r02n/c4.json').read().splitlines()[-1]); print('c4', d['value'], d['e2e']['value'], d['per_gpu']['restart_ms'], d['verified']['ok'])"
