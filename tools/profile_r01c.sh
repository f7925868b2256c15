#!/bin/bash
# ncu evidence, round 1 (third pass: 64 MiB windows, hash+copy snapshot).  One GPU.
NCU=/usr/local/cuda/bin/ncu
OUT=gpurun_out/r01c
mkdir -p $OUT
# full sets of the hot kernels inside the C4 drain/refill on an 8 GiB state
for k in k1_chunk_crc k_pack_records k_scatter_records; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$k -s 40 -c 1 \
    -o $OUT/prof_$k python bench.py --footprint-gib 8 --steps 1 --warmup 1 \
    --no-cpu-baseline --no-incremental --no-stall > $OUT/prof_$k.log 2>&1
done
# the fused hash+copy kernel of the stall-reduced drain (its first K1 launch)
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k1_chunk_crc -c 1 \
  -o $OUT/prof_k1_hash_copy python tools/stall_probe.py 8 > $OUT/prof_k1_hash_copy.log 2>&1
# launch list of the default bench command (setup + warmup + one step)
timeout 2400 $NCU --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
  --no-incremental --no-stall > $OUT/launches_bench.log 2>&1
ls -la $OUT
