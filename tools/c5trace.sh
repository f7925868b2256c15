CRAC_TRACE=1 timeout 600 python bench.py --workload c5 --steps 1 --warmup 0 --c5-footprint-gib 64 > gpurun_out/c5t.json 2> gpurun_out/c5t.err
