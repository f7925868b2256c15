# round 2cf: C3 checkpoint regression hunt -- commit 07e34f4 (before the streamed host copies and the split-drain
# event fix, built in .abtree) against the current build, same box, alternating
mkdir -p gpurun_out/r02cf
for rep in 1 2; do
for t in old new; do
if [ $t = old ]; then d=.abtree; else d=.; fi
(cd $d && timeout 600 python bench.py --workload c3 --no-stall --no-cpu-baseline --no-verify) > gpurun_out/r02cf/c3_${t}_$rep.json 2>gpurun_out/r02cf/c3_${t}_$rep.err
python -c "
import json; d=json.loads(open('gpurun_out/r02cf/c3_${t}_$rep.json').read().splitlines()[-1]); r=d['roofline']
print('c3 $t', d['value'], d['per_gpu']['checkpoint_ms'], d['per_gpu']['restart_ms'], r['d2h_GBps_per_step'])"
done
done
