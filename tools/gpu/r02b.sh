# round 2b: dirty-key lane (tests + C5 hash-only rate), UVM populate probe
mkdir -p gpurun_out/r02b
nproc; lscpu | grep -i "model name\|socket\|numa node(s)\|^CPU(s)"
python -m pytest tests -x -q -m gpu > gpurun_out/r02b/gputests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02b/gputests.log
timeout 300 ./tools/probe/probe_uvm3 16 > gpurun_out/r02b/probe_uvm3.txt 2>&1; echo "probe rc=$?"
cat gpurun_out/r02b/probe_uvm3.txt
python bench.py --workload c5 --steps 3 --warmup 2 --no-stall > gpurun_out/r02b/bench_c5.json 2> gpurun_out/r02b/bench_c5.err; echo "c5 rc=$?"
python bench.py --steps 3 --warmup 3 --no-stall --no-cpu-baseline > gpurun_out/r02b/bench_c4.json 2> gpurun_out/r02b/bench_c4.err; echo "c4 rc=$?"
