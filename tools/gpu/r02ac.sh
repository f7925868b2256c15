# round 2ac: aligned direct pieces after an exact head; PCIe peaks re-measured after the loop
mkdir -p gpurun_out/r02ac
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x > gpurun_out/r02ac/gputests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02ac/gputests.log
for rep in 1 2; do
timeout 900 python bench.py --steps 3 --warmup 2 --no-stall --no-cpu-baseline --no-incremental > gpurun_out/r02ac/c4_$rep.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/r02ac/c4_$rep.json').read().splitlines()[-1]); r=d['roofline']; print('c4', d['value'], d['e2e']['value'], d['per_gpu']['restart_ms'], r['frac'], r['h2d_GBps_per_step'], r['d2h_peak_GBps'], r['h2d_peak_GBps'], d['verified']['ok'])"
done
timeout 600 python bench.py --workload c2 --steps 8 --warmup 3 --no-stall --no-cpu-baseline > gpurun_out/r02ac/c2.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02ac/c2.json').read().splitlines()[-1]); print('c2', d['value'], d['e2e']['value'], d['per_gpu']['restart_ms'], d['roofline']['frac'])"
