#!/bin/bash
# K1 rows experiment + traced bench (run under gpurun)
for r in 4 8 16; do
  CRAC_K1_ROWS=$r timeout 300 python bench.py --footprint-gib 32 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/k1_rows_$r.json 2> gpurun_out/k1_rows_$r.err
done
CRAC_TRACE=1 timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_trace.json 2> gpurun_out/bench_trace.err
