# round 2aq: K1 waves over all SMs during the drain (pack on a high-priority stream) vs 132 persistent CTAs
mkdir -p gpurun_out/r02aq
for rep in 1 2; do for wv in 0 4 8; do
CRAC_K1_WAVES=$wv timeout 900 python bench.py --steps 3 --warmup 2 --no-stall --no-cpu-baseline --no-incremental --no-verify > gpurun_out/r02aq/c4_${wv}_$rep.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/r02aq/c4_${wv}_$rep.json').read().splitlines()[-1]); r=d['roofline']; k=r['kernels']['k1_chunk_crc']; print('waves=$wv', d['value'], d['per_gpu']['checkpoint_ms'], k['achieved'], k['frac'], r['d2h_GBps_per_step'])"
done; done
