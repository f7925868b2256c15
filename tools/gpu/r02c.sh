# round 2c: first GPU pass of this round: full GPU suite (dirty key, BASELINE-size parity), C4/C5 bench, UVM populate probe
mkdir -p gpurun_out/r02c
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/r02c/gputests.log 2>&1; echo "tests rc=$?"
tail -25 gpurun_out/r02c/gputests.log
timeout 300 ./tools/probe/probe_uvm3 16 > gpurun_out/r02c/probe_uvm3.txt 2>&1; echo "probe rc=$?"
cat gpurun_out/r02c/probe_uvm3.txt
timeout 600 python bench.py --workload c5 --steps 3 --warmup 3 --no-stall > gpurun_out/r02c/bench_c5.json 2> gpurun_out/r02c/bench_c5.err; echo "c5 rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02c/bench_c4.json 2> gpurun_out/r02c/bench_c4.err; echo "c4 rc=$?"
tail -c 1500 gpurun_out/r02c/bench_c4.json
