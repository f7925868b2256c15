# round 2bb: does the drain mode before an incremental drain change it?  C5 after a ring drain (CRAC_DIRECT=refill) against a direct one (both), alternating
mkdir -p gpurun_out/r02bb
for rep in 1 2; do
for m in refill both; do
CRAC_DIRECT=$m timeout 900 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline --no-verify --no-stall > gpurun_out/r02bb/c5_${m}_$rep.json 2>gpurun_out/r02bb/c5_${m}_$rep.err; python -c "
import json; d=json.loads(open('gpurun_out/r02bb/c5_${m}_$rep.json').read().splitlines()[-1]); i=d['incremental']
print('c5 direct=$m', [(k, v['drain_ms'], v['drain_roofline_ms'], round(v['drain_roofline_ms']/v['drain_ms'],3), v['hash_frac_of_hbm']) for k,v in i.items()])"
done
done
