# round 2k: early windows only into mapped arenas, single-run cold premap; C2 / C3 bench; split-drain ncu
mkdir -p gpurun_out/r02k gpurun_out/r02p
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_barrier.py -x -q > gpurun_out/r02k/gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02k/gputests.log
timeout 600 python bench.py --workload c2 --steps 5 --warmup 3 --no-stall > gpurun_out/r02k/bench_c2.json 2> gpurun_out/r02k/bench_c2.err; echo "c2 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02k/bench_c2.json').read().splitlines()[-1]); print(d['value'], d['e2e']['value'], json.dumps(d['per_gpu']), d['roofline']['frac'])"
CRAC_TRACE=1 timeout 600 python bench.py --workload c2 --steps 2 --warmup 2 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02k/c2_trace.json 2> gpurun_out/r02k/c2_trace.err; echo "trace rc=$?"
timeout 600 python bench.py --workload c3 --steps 3 --warmup 2 --no-stall > gpurun_out/r02k/bench_c3.json 2> gpurun_out/r02k/bench_c3.err; echo "c3 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02k/bench_c3.json').read().splitlines()[-1]); print(d['value'], d['e2e']['value'], json.dumps(d['per_gpu']), json.dumps({k: d['roofline'][k] for k in ('bound','achieved','peak','frac','floor_ms')}))"
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on \
  --kernel-name-base demangled -k "regex:k1_chunk_crc<\(int\)4, \(int\)4" -s 1 -c 1 \
  -o gpurun_out/r02p/prof_k1_split python bench.py --workload c5 --c5-footprint-gib 16 --steps 1 --warmup 1 \
  --no-stall > gpurun_out/r02p/prof_k1_split.log 2>&1; echo "ncu split rc=$?"
