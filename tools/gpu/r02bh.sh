# round 2bh: is the C4 refill scatter's in-situ span the cold tail map beside it?  default (8 GiB head, tail mapped on
# a thread) against CRAC_COLD_HEAD_MIB=0 (whole arena mapped before the copies)
mkdir -p gpurun_out/r02bh
for h in default 0; do
if [ $h = 0 ]; then export CRAC_COLD_HEAD_MIB=0; else unset CRAC_COLD_HEAD_MIB; fi
timeout 900 python bench.py --steps 2 --warmup 3 --no-stall --no-cpu-baseline --no-incremental --no-verify > gpurun_out/r02bh/c4_head_$h.json 2>gpurun_out/r02bh/c4_head_$h.err
python -c "
import json; d=json.loads(open('gpurun_out/r02bh/c4_head_$h.json').read().splitlines()[-1]); k=d['roofline']['kernels']
print('head=$h', d['value'], d['per_gpu']['restart_ms'], 'scatter', k.get('k_scatter_records',{}).get('avg_launch_ms'), k.get('k_scatter_records',{}).get('launches'), 'verify', k.get('k1_chunk_crc (refill verify)',{}).get('frac'))"
done
