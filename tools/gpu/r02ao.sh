# round 2ao: TMA (cp.async.bulk) writers for the split incremental drain: parity + C5 A/B
mkdir -p gpurun_out/r02ao
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x -k "alternative or incremental or dirty or forged or split" > gpurun_out/r02ao/gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02ao/gputests.log
CRAC_WRITER_TMA=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -q -x > gpurun_out/r02ao/gputests_tma.log 2>&1; echo "tests(tma) rc=$?"; tail -2 gpurun_out/r02ao/gputests_tma.log
for rep in 1 2; do for t in 1 0; do
CRAC_WRITER_TMA=$t timeout 900 python bench.py --workload c5 --steps 3 --warmup 2 --no-stall --no-verify > gpurun_out/r02ao/c5_${t}_$rep.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/r02ao/c5_${t}_$rep.json').read().splitlines()[-1]); r=d['incremental']; print('tma=$t', {k: (v['drain_ms'], v['drain_roofline_ms']) for k,v in r.items()})"
done; done
CRAC_WRITER_TMA=1 timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_paths.py > gpurun_out/r02ao/racecheck_tma.txt 2>&1; echo "racecheck rc=$?"; tail -1 gpurun_out/r02ao/racecheck_tma.txt
CRAC_WRITER_TMA=1 timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_paths.py > gpurun_out/r02ao/memcheck_tma.txt 2>&1; echo "memcheck rc=$?"; tail -1 gpurun_out/r02ao/memcheck_tma.txt
