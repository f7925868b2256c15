#!/bin/bash
# ncu evidence, round 1 (fourth pass: direct runs + edge pack/scatter, host-run C3 path).
NCU=/usr/local/cuda/bin/ncu
OUT=gpurun_out/r01d
mkdir -p $OUT
# full sets of the hot kernels inside the C4 drain/refill on an 8 GiB state
for k in k1_chunk_crc k_pack_records k_scatter_records; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$k -s 40 -c 1 \
    -o $OUT/prof_$k python bench.py --footprint-gib 8 --steps 1 --warmup 1 \
    --no-cpu-baseline --no-incremental --no-stall > $OUT/prof_$k.log 2>&1
done
# launch list of the default bench command (setup + warmup + one step)
timeout 3000 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
  --no-incremental --no-stall > $OUT/launches_bench.log 2>&1
ls -la $OUT
