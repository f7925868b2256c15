#!/bin/bash
# ncu evidence, round 1 (second pass, after the kernel rework).  One GPU.
NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out/r01b
# full sets of the hot kernels on a 4 GiB C4 state (K1 in-drain, pack, scatter)
for k in k1_chunk_crc k_pack_records k_scatter_records; do
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o gpurun_out/r01b/prof_$k python bench.py --footprint-gib 4 --steps 1 --warmup 1 \
    --no-cpu-baseline --no-incremental > gpurun_out/r01b/prof_$k.log 2>&1
done
# the fused incremental hash+drain kernel (C5 shape, 8 GiB, 1 % dirty)
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k1_chunk_crc -s 4 -c 1 \
  -o gpurun_out/r01b/prof_k1_fused_drain python bench.py --workload c5 --c5-footprint-gib 8 \
  --steps 1 --warmup 0 > gpurun_out/r01b/prof_k1_fused.log 2>&1
# launch list of the default bench command (setup + first step)
timeout 2000 $NCU --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
  --log-file gpurun_out/r01b/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
  > gpurun_out/r01b/launches_bench.log 2>&1
ls -la gpurun_out/r01b
