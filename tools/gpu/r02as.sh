# round 2as: cold refill head-start buffer (early windows outside the arena while it is mapped)
mkdir -p gpurun_out/r02as
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r02as/gputests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02as/gputests.log
for rep in 1 2; do for cw in 96 0; do
CRAC_COLD_WINDOWS=$cw timeout 900 python bench.py --steps 3 --warmup 2 --no-stall --no-cpu-baseline --no-incremental > gpurun_out/r02as/c4_${cw}_$rep.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/r02as/c4_${cw}_$rep.json').read().splitlines()[-1]); print('c4 cold_windows=$cw', d['value'], d['e2e']['value'], d['per_gpu']['restart_ms'], d['per_gpu']['warm_restart']['restart_ms'], d['roofline']['frac'], d['verified']['ok'])"
done; done
for cw in 96 0; do CRAC_COLD_WINDOWS=$cw timeout 600 python bench.py --workload c2 --steps 8 --warmup 3 --no-stall --no-cpu-baseline > gpurun_out/r02as/c2_$cw.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02as/c2_$cw.json').read().splitlines()[-1]); print('c2 cold_windows=$cw', d['value'], d['e2e']['value'], d['per_gpu']['restart_ms'], d['verified']['ok'])"; done
