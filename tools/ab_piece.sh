#!/bin/bash
# Ring window D2H/H2D piece size A/B on C4, 3 alternating rounds.
for round in 1 2 3; do
for mib in 16 32 64; do
  CRAC_COPY_CHUNK_MIB=$mib timeout 900 python bench.py --no-cpu-baseline --no-incremental --no-stall --steps 3 --warmup 2 > /tmp/out.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('/tmp/out.json')); print('piece', sys.argv[1], '|', d['per_gpu']['checkpoint_GBps'], d['per_gpu']['restart_GBps'], d['value'], d['pcie_roofline']['d2h_peak_GBps'])" "$mib"
done; done
