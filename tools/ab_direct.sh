mkdir -p gpurun_out/ab
for cfg in "CRAC_DIRECT=0" "CRAC_DIRECT=both" "CRAC_DIRECT=both CRAC_DIRECT_PIECE_MIB=16" "CRAC_DIRECT=both CRAC_DIRECT_PIECE_MIB=32" "CRAC_DIRECT=refill"; do
  env $cfg timeout 900 python bench.py --no-cpu-baseline --no-incremental --no-stall --steps 3 --warmup 2 > gpurun_out/ab/out.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/ab/out.json')); print(sys.argv[1], d['value'], d['per_gpu']['checkpoint_GBps'], d['per_gpu']['restart_GBps'], d['pcie_roofline']['d2h_peak_GBps'], d['pcie_roofline']['h2d_peak_GBps'])" "$cfg"
done
