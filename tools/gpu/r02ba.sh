# round 2ba: drain through the ring (CRAC_DIRECT=refill) against direct D2H (both) with K1 leaving 16 or 4 SMs, C4, alternating
mkdir -p gpurun_out/r02ba
for rep in 1 2; do
for v in "refill 16" "both 16" "both 4"; do
set -- $v
CRAC_DIRECT=$1 CRAC_K1_SPARE_SMS=$2 timeout 900 python bench.py --steps 3 --warmup 3 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02ba/c4_$1_$2_$rep.json 2>gpurun_out/r02ba/c4_$1_$2_$rep.err; python -c "
import json; d=json.loads(open('gpurun_out/r02ba/c4_$1_$2_$rep.json').read().splitlines()[-1]); r=d['roofline']; k=r['kernels']; i=d.get('incremental',{})
print('direct=$1 spare=$2', d['value'], d['e2e']['value'], d['per_gpu']['checkpoint_ms'], d['per_gpu']['restart_ms'], r['d2h_GBps_per_step'], 'K1', k['k1_chunk_crc']['frac'], 'inc1%', i.get('drain_1pct',{}).get('ms'), 'hash_only', i.get('hash_only',{}).get('frac_of_hbm'))"
done
done
