# round 2bi: C2 refill verify in batches as windows land (CRAC_VERIFY_SPLIT=4, default) against one batch at the end (=1), alternating
mkdir -p gpurun_out/r02bi
for rep in 1 2 3; do
for v in 4 1; do
CRAC_VERIFY_SPLIT=$v timeout 600 python bench.py --workload c2 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02bi/c2_split${v}_$rep.json 2>gpurun_out/r02bi/c2_split${v}_$rep.err
python -c "
import json; d=json.loads(open('gpurun_out/r02bi/c2_split${v}_$rep.json').read().splitlines()[-1]); k=d['roofline']['kernels'].get('k1_chunk_crc (refill verify)',{})
print('split=$v', d['value'], d['e2e']['value'], d['per_gpu']['checkpoint_ms'], d['per_gpu']['restart_ms'], d['roofline']['frac'], 'verify launches', k.get('launches'), k.get('avg_launch_ms'))"
done
done
