# round 2j: C2 after the host_pre fix (+ trace), parity suite, then the r02 ncu profile set
mkdir -p gpurun_out/r02j
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q > gpurun_out/r02j/gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02j/gputests.log
timeout 600 python bench.py --workload c2 --steps 5 --warmup 3 --no-stall > gpurun_out/r02j/bench_c2.json 2> gpurun_out/r02j/bench_c2.err; echo "c2 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02j/bench_c2.json').read().splitlines()[-1]); print(d['value'], d['e2e']['value'], json.dumps(d['per_gpu']), d['roofline']['frac'])"
CRAC_TRACE=1 timeout 600 python bench.py --workload c2 --steps 2 --warmup 2 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02j/c2_trace.json 2> gpurun_out/r02j/c2_trace.err; echo "trace rc=$?"
bash tools/profile_r02.sh > gpurun_out/r02j/profile.log 2>&1; echo "profile rc=$?"
tail -5 gpurun_out/r02j/profile.log
