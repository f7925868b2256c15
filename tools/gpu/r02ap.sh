# round 2ap: final build: full GPU suite, smoke, default bench line, reference arm, C5
mkdir -p gpurun_out/r02ap
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r02ap/gputests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02ap/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ap/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02ap/smoke.log
timeout 900 python bench.py > gpurun_out/r02ap/bench_c4.json 2> gpurun_out/r02ap/bench_c4.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02ap/bench_c4.json').read().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['verified']['ok'], d['gpu_launches'], d['clocks'], d['incremental']['hash_only']['frac_of_hbm'])"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02ap/bench_reference.json 2> gpurun_out/r02ap/bench_reference.err; echo "ref rc=$?"; tail -c 300 gpurun_out/r02ap/bench_reference.json
timeout 900 python bench.py --workload c5 > gpurun_out/r02ap/bench_c5.json 2> gpurun_out/r02ap/bench_c5.err; echo "c5 rc=$?"
