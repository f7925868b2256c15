#!/bin/bash
# Every bench workload once on one GPU; JSON lines to $OUT (default gpurun_out/all).
OUT=${OUT:-gpurun_out/all}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
timeout 900 python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 600 python bench.py --workload c2 > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 600 python bench.py --workload c3 > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 900 python bench.py --workload c5 > $OUT/bench_c5.json 2> $OUT/bench_c5.err
timeout 900 python bench.py --workload file --steps 2 --warmup 1 > $OUT/bench_file.json 2> $OUT/bench_file.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
for f in $OUT/bench_*.json; do echo "== $f"; head -c 600 $f; echo; done
