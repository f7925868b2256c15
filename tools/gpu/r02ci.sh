# round 2ci: run-to-run spread of the default bench line on the last build (3 back-to-back runs)
mkdir -p gpurun_out/r02ci
for rep in 1 2 3; do
timeout 900 python bench.py > gpurun_out/r02ci/bench_c4_$rep.json 2> gpurun_out/r02ci/bench_c4_$rep.err
python -c "
import json; d=json.loads(open('gpurun_out/r02ci/bench_c4_$rep.json').read().splitlines()[-1]); r=d['roofline']
print('c4 run $rep', d['value'], d['e2e']['value'], r['frac'], d['per_gpu']['checkpoint_ms'], d['per_gpu']['restart_ms'], r['d2h_peak_GBps'], 'K1', r['kernels']['k1_chunk_crc']['frac'], 'verified', d['verified']['ok'], d['clocks']['reasons'])"
done
