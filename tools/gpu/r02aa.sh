# round 2aa: final-build full GPU suite + smoke, then every bench workload
mkdir -p gpurun_out/r02aa
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r02aa/gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02aa/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02aa/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02aa/smoke.log
OUT=gpurun_out/r02aa/all bash tools/bench_all.sh > gpurun_out/r02aa/all.log 2>&1; echo "all rc=$?"
for w in c4 c2 c3 c5 file reference; do python -c "
import json,sys
d=json.loads(open('gpurun_out/r02aa/all/bench_$w.json').read().splitlines()[-1])
print('$w', d.get('value'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('verified') or {}).get('ok'))
" 2>&1 | tail -1; done
