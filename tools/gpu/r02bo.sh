# round 2bo: C4 cold restart with the early ring windows (default) against none (CRAC_COLD_FULLMAP=0: the arena mapped
# from the active set after the parse, direct runs from the first byte), alternating
mkdir -p gpurun_out/r02bo
for rep in 1 2; do
for m in default nofull; do
if [ $m = nofull ]; then export CRAC_COLD_FULLMAP=0; else unset CRAC_COLD_FULLMAP; fi
timeout 900 python bench.py --steps 3 --warmup 3 --no-stall --no-cpu-baseline --no-incremental --no-verify > gpurun_out/r02bo/c4_${m}_$rep.json 2>gpurun_out/r02bo/c4_${m}_$rep.err
python -c "
import json; d=json.loads(open('gpurun_out/r02bo/c4_${m}_$rep.json').read().splitlines()[-1]); r=d['roofline']; k=r['kernels']
print('$m', d['value'], d['e2e']['value'], d['per_gpu']['checkpoint_ms'], d['per_gpu']['restart_ms'], r['h2d_GBps_per_step'], r['h2d_peak_GBps'], 'scatter', k.get('k_scatter_records',{}).get('launches'), k.get('k_scatter_records',{}).get('avg_launch_ms'))"
done
done
