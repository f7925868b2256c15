#!/bin/bash
# ncu evidence, round 1 (fourth pass: direct runs + edge pack/scatter, host-run C3 path).
# One GPU.  Outputs gpurun_out/r01d; summarise with tools/ncu_summary.py.
NCU=/usr/local/cuda/bin/ncu
OUT=gpurun_out/r01d
mkdir -p $OUT
BENCH8="python bench.py --footprint-gib 8 --steps 1 --warmup 1 --no-cpu-baseline --no-incremental --no-stall"
# K1 of the timed drain (8 GiB: warmup drain 1 + warmup refill verify 16 launches before it)
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k1_chunk_crc -s 17 -c 1 \
  -o $OUT/prof_k1_drain $BENCH8 > $OUT/prof_k1_drain.log 2>&1
# a refill-verify K1 batch (512 MiB)
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k1_chunk_crc -s 1 -c 1 \
  -o $OUT/prof_k1_chunk_crc $BENCH8 > $OUT/prof_k1_chunk_crc.log 2>&1
for k in k_pack_records k_scatter_records; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$k -s 40 -c 1 \
    -o $OUT/prof_$k $BENCH8 > $OUT/prof_$k.log 2>&1
done
# launch list of the default bench command (setup + warmup + one step).  At the
# default 120 GiB the process is OOM-killed under ncu on this 196 GB host, so
# the list is taken at 96 GiB (same regions, same code path).
timeout 3000 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv \
  --log-file $OUT/launches.csv python bench.py --footprint-gib 96 --steps 1 --warmup 1 \
  --no-cpu-baseline --no-incremental --no-stall > $OUT/launches_bench.log 2>&1
echo "launch run exit $?" >> $OUT/launches_bench.log
ls -la $OUT
