# round 2bd: streamed checkpoint_to_file: persistence GPU tests, then the file workload streamed vs drain-then-write (the default; this run set CRAC_FILE_NO_STREAM=1 when streaming was the default), alternating
mkdir -p gpurun_out/r02bd
timeout 900 python -m pytest tests/test_gpu_persistence.py -x -q > gpurun_out/r02bd/persist.log 2>&1; tail -3 gpurun_out/r02bd/persist.log
for rep in 1 2; do
for m in stream plain; do
if [ $m = plain ]; then export CRAC_FILE_NO_STREAM=1; else unset CRAC_FILE_NO_STREAM; fi
timeout 900 python bench.py --workload file --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02bd/file_${m}_$rep.json 2>gpurun_out/r02bd/file_${m}_$rep.err; python -c "
import json; d=json.loads(open('gpurun_out/r02bd/file_${m}_$rep.json').read().splitlines()[-1]); p=d['per_gpu']; r=d['roofline'] or {}
print('file $m', d['value'], p['checkpoint_to_file_s'], p['restart_from_file_s'], p['phases_ms'], p.get('streamed_bytes'), r.get('frac'))"
done
done
