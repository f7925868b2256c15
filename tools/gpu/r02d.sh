# round 2d: barrier GPU tests, K1 key-lane depth experiment, C5 with the 8-row key variants
mkdir -p gpurun_out/r02d
timeout 600 python -m pytest tests/test_gpu_barrier.py tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q > gpurun_out/r02d/gputests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r02d/gputests.log
timeout 600 python tools/exp_k1_key.py > gpurun_out/r02d/k1_key.txt 2>&1; echo "exp rc=$?"
cat gpurun_out/r02d/k1_key.txt
timeout 600 python bench.py --workload c5 --steps 3 --warmup 2 --no-stall > gpurun_out/r02d/bench_c5.json 2> gpurun_out/r02d/bench_c5.err; echo "c5 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02d/bench_c5.json').read().splitlines()[-1]); print(json.dumps(d['incremental']))"
