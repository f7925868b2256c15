# round 2cg: streamed host copies now opt-in (CRAC_HOST_NT=1); C3 with it off (default) / on against the pre-change build
mkdir -p gpurun_out/r02cg
for rep in 1 2; do
for t in old off on; do
d=.; env=""
if [ $t = old ]; then d=.abtree; fi
if [ $t = on ]; then env="CRAC_HOST_NT=1"; fi
(cd $d && env $env timeout 600 python bench.py --workload c3 --no-stall --no-cpu-baseline --no-verify) > gpurun_out/r02cg/c3_${t}_$rep.json 2>gpurun_out/r02cg/c3_${t}_$rep.err
python -c "
import json; d=json.loads(open('gpurun_out/r02cg/c3_${t}_$rep.json').read().splitlines()[-1]); r=d['roofline']
print('c3 $t', d['value'], d['per_gpu']['checkpoint_ms'], d['per_gpu']['restart_ms'], r['d2h_GBps_per_step'])"
done
done
