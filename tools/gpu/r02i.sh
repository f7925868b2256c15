# round 2i: engine stress restatement (bounded run, progress), sanitizers on every path,
# parity suites (pinned host path, early refill windows), C2 bench
mkdir -p gpurun_out/r02i
timeout 400 ./tools/probe/engine_stress 100 > gpurun_out/r02i/engine_stress_100.txt 2>&1; echo "stress rc=$?"
tail -8 gpurun_out/r02i/engine_stress_100.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_paths.py > gpurun_out/r02i/sanitizer_$tool.txt 2>&1; echo "$tool rc=$?"
  tail -2 gpurun_out/r02i/sanitizer_$tool.txt
done
timeout 1200 python -m pytest tests -x -q -m gpu --deselect tests/test_engine_stress.py::test_engine_stress_restated_on_b200 > gpurun_out/r02i/gputests.log 2>&1; echo "tests rc=$?"
tail -4 gpurun_out/r02i/gputests.log
timeout 600 python bench.py --workload c2 --steps 5 --warmup 3 --no-stall > gpurun_out/r02i/bench_c2.json 2> gpurun_out/r02i/bench_c2.err; echo "c2 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02i/bench_c2.json').read().splitlines()[-1]); print(d['value'], d['e2e']['value'], json.dumps(d['per_gpu']), d['roofline']['frac'])"
