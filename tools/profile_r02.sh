#!/bin/bash
# ncu evidence, round 2: paired-chain K1 (drain with the key lane; refill verify
# CRC only), pack / scatter, the split incremental drain kernel, and the launch
# list of the bench command.  One GPU.  Outputs gpurun_out/r02p; summarise with
# tools/ncu_summary.py gpurun_out/r02p profiles/r02.
NCU=/usr/local/cuda/bin/ncu
OUT=gpurun_out/r02p
mkdir -p $OUT
BENCH8="python bench.py --footprint-gib 8 --steps 1 --warmup 1 --no-cpu-baseline --no-incremental --no-stall --no-verify --no-cold"
# launch order at 8 GiB: warmup drain K1 (1), warmup refill verify K1 (4 x 2 GiB),
# timed drain K1, timed refill verify ...
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k1_chunk_crc -s 5 -c 1 \
  -o $OUT/prof_k1_drain $BENCH8 > $OUT/prof_k1_drain.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k1_chunk_crc -s 1 -c 1 \
  -o $OUT/prof_k1_chunk_crc $BENCH8 > $OUT/prof_k1_chunk_crc.log 2>&1
for k in k_pack_records k_scatter_records; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$k -s 40 -c 1 \
    -o $OUT/prof_$k $BENCH8 > $OUT/prof_$k.log 2>&1
done
# the split incremental drain (C5 shape at 16 GiB, 5 % dirty)
timeout 900 $NCU --set full --clock-control none --import-source on \
  --kernel-name-base demangled -k "regex:k1_chunk_crc<\(int\)4, \(int\)4" -s 1 -c 1 \
  -o $OUT/prof_k1_split python bench.py --workload c5 --c5-footprint-gib 16 --steps 1 --warmup 1 \
  --no-stall > $OUT/prof_k1_split.log 2>&1
timeout 3000 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv \
  --log-file $OUT/launches.csv python bench.py --footprint-gib 96 --steps 1 --warmup 1 \
  --no-cpu-baseline --no-incremental --no-stall --no-verify --no-cold > $OUT/launches_bench.log 2>&1
echo "launch run exit $?" >> $OUT/launches_bench.log
ls -la $OUT
