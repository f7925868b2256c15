# round 2g: K1 paired chains experiment (+parity), UVM populate probe 4, C4 bench with the lazy premap (cold restart)
mkdir -p gpurun_out/r02g
timeout 900 python tools/exp_k1_key.py > gpurun_out/r02g/k1_key.txt 2>&1; echo "exp rc=$?"
cat gpurun_out/r02g/k1_key.txt
timeout 300 ./tools/probe/probe_uvm4 16 > gpurun_out/r02g/probe_uvm4.txt 2>&1; echo "probe rc=$?"
cat gpurun_out/r02g/probe_uvm4.txt
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q > gpurun_out/r02g/gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02g/gputests.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-stall --no-cpu-baseline > gpurun_out/r02g/bench_c4.json 2> gpurun_out/r02g/bench_c4.err; echo "c4 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02g/bench_c4.json').read().splitlines()[-1]); print(d['value'], d['e2e']['value'], json.dumps(d['per_gpu']), d['roofline']['frac'])"
