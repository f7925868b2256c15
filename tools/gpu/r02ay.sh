# round 2ay: drain with direct D2H from the allocations (CRAC_DIRECT=both) vs through the ring (default), C4; plus a C2 phase trace
mkdir -p gpurun_out/r02ay
CRAC_TRACE=1 timeout 600 python bench.py --workload c2 --steps 2 --warmup 2 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02ay/c2_trace.json 2> gpurun_out/r02ay/c2_trace.err
for rep in 1 2; do
for d in refill both; do
CRAC_DIRECT=$d timeout 900 python bench.py --steps 3 --warmup 2 --no-stall --no-cpu-baseline --no-incremental --no-verify > gpurun_out/r02ay/c4_${d}_$rep.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02ay/c4_${d}_$rep.json').read().splitlines()[-1]); r=d['roofline']; print('c4 direct=$d', d['value'], d['e2e']['value'], d['per_gpu']['checkpoint_ms'], d['per_gpu']['restart_ms'], r['d2h_GBps_per_step'], r['kernels'].get('k_pack_records',{}).get('launches'))"
done
done
