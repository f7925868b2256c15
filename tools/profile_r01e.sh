#!/bin/bash
# ncu evidence for the kernels added late in round 1: the split incremental
# drain (K1 mode 4) and the 512-thread pack.  One GPU.
NCU=/usr/local/cuda/bin/ncu
OUT=gpurun_out/r01e
mkdir -p $OUT
timeout 900 $NCU --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k1_chunk_crc<\\(int\\)16, \\(int\\)4>" -c 1 -o $OUT/prof_k1_split_drain \
  python bench.py --workload c5 --c5-footprint-gib 8 --steps 1 --warmup 0 --no-stall \
  > $OUT/prof_k1_split_drain.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_pack_records -s 40 -c 1 \
  -o $OUT/prof_k_pack_records python bench.py --footprint-gib 8 --steps 1 --warmup 1 \
  --no-cpu-baseline --no-incremental --no-stall > $OUT/prof_k_pack_records.log 2>&1
ls -la $OUT
