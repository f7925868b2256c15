# round 2at: final build: full GPU suite, smoke, every bench workload, reference arm
mkdir -p gpurun_out/r02at
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r02at/gputests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02at/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02at/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02at/smoke.log
OUT=gpurun_out/r02at/all bash tools/bench_all.sh > gpurun_out/r02at/all.log 2>&1; echo "all rc=$?"
for w in c4 c2 c3 c5 file reference; do python -c "
import json
d=json.loads(open('gpurun_out/r02at/all/bench_$w.json').read().splitlines()[-1])
print('$w', d.get('value'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('verified') or {}).get('ok'))
" 2>&1 | tail -1; done
