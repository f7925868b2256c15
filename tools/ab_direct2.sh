#!/bin/bash
# Drain/refill A/B of the direct runs, 3 alternating rounds per mode (C4, 120 GiB).
mkdir -p gpurun_out/ab2
for round in 1 2 3; do
for cfg in "CRAC_DIRECT=0" "CRAC_DIRECT=refill" "CRAC_DIRECT=both" "CRAC_DIRECT=both CRAC_DIRECT_PIECE_MIB=16"; do
  env $cfg timeout 900 python bench.py --no-cpu-baseline --no-incremental --no-stall --steps 3 --warmup 2 > gpurun_out/ab2/out.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/ab2/out.json')); print(sys.argv[1], '|', d['per_gpu']['checkpoint_GBps'], d['per_gpu']['restart_GBps'], d['value'], d['pcie_roofline']['d2h_peak_GBps'])" "$cfg"
done; done
