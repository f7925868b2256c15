#!/bin/bash
# ncu evidence for round 1 (run under gpurun; one GPU).
set -x
NCU=/usr/local/cuda/bin/ncu
# 1) launch list of the bench command (device time per launch, cold/serialised)
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
  > gpurun_out/launches_bench.log 2>&1
# 2) full sets for the three hot kernels on a 4 GiB state
for k in k1_chunk_crc k_pack_records k_scatter_records; do
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/prof_$k python bench.py --footprint-gib 4 --steps 1 --warmup 1 \
    --no-cpu-baseline --no-incremental > gpurun_out/prof_$k.log 2>&1
done
ls -la gpurun_out
