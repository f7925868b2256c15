set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -x -q -m gpu > gpurun_out/r02a/gputests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r02a/gputests.log
python bench.py --steps 5 --warmup 3 > gpurun_out/r02a/bench_c4.json 2> gpurun_out/r02a/bench_c4.err; echo "bench rc=$?"
python bench.py --workload c3 --steps 3 --warmup 2 --no-stall > gpurun_out/r02a/bench_c3.json 2> gpurun_out/r02a/bench_c3.err
CRAC_TRACE=1 python bench.py --workload c3 --steps 1 --warmup 1 --no-stall --no-cpu-baseline --no-cold > gpurun_out/r02a/c3_trace.json 2> gpurun_out/r02a/c3_trace.err
tail -c 600 gpurun_out/r02a/bench_c4.json
