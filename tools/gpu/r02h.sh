# round 2h: full GPU suite (paired K1 default, writers-last split drain + occupancy fallback,
# bounded quiesce drain, engine stress restatement), compute-sanitizer on every kernel path,
# C4 / C5 / C3 bench
mkdir -p gpurun_out/r02h
timeout 1800 python -m pytest tests -x -q -m gpu --durations=10 > gpurun_out/r02h/gputests.log 2>&1; echo "tests rc=$?"
tail -16 gpurun_out/r02h/gputests.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_paths.py > gpurun_out/r02h/sanitizer_$tool.txt 2>&1; echo "$tool rc=$?"
  tail -3 gpurun_out/r02h/sanitizer_$tool.txt
done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02h/bench_c4.json 2> gpurun_out/r02h/bench_c4.err; echo "c4 rc=$?"
timeout 600 python bench.py --workload c5 --steps 3 --warmup 2 --no-stall > gpurun_out/r02h/bench_c5.json 2> gpurun_out/r02h/bench_c5.err; echo "c5 rc=$?"
timeout 600 python bench.py --workload c3 --steps 3 --warmup 2 --no-stall > gpurun_out/r02h/bench_c3.json 2> gpurun_out/r02h/bench_c3.err; echo "c3 rc=$?"
