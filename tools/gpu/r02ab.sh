# round 2ab: refill direct runs to the payloads' exact ends, scatter launched only where needed
mkdir -p gpurun_out/r02ab
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r02ab/gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02ab/gputests.log
timeout 900 python bench.py --steps 3 --warmup 2 --no-stall --no-cpu-baseline > gpurun_out/r02ab/c4.json 2>/dev/null; echo "c4 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02ab/c4.json').read().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['per_gpu']['restart_ms'], d['roofline']['frac'], d['verified']['ok'], d['gpu_launches']); print({k:(v['launches'], v['avg_launch_ms'], v['achieved']) for k,v in d['roofline']['kernels'].items()})"
for rep in 1 2; do timeout 600 python bench.py --workload c2 --steps 8 --warmup 3 --no-stall --no-cpu-baseline > gpurun_out/r02ab/c2_$rep.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02ab/c2_$rep.json').read().splitlines()[-1]); print('c2', d['value'], d['e2e']['value'], d['per_gpu']['restart_ms'], d['roofline']['frac'])"; done
