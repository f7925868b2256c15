# round 2bz: the async drain's window-event fix (checkpoint_finish with stats after a checkpoint_begin without them read
# events never created): the crashing orders first, then the full GPU suite, then C3 with the NT host copy on / off
mkdir -p gpurun_out/r02bz
A="tests/test_gpu_parity.py::test_pinned_payloads_move_on_the_host_and_match_reference[all-shadow]"
B="tests/test_gpu_parity.py::test_async_drain_with_managed_runs_matches_reference[64]"
timeout 300 python -X faulthandler -m pytest -x -q "$A" "$B" > gpurun_out/r02bz/ab.log 2>&1; echo "A,B exit $?: $(tail -1 gpurun_out/r02bz/ab.log)"
timeout 600 python -X faulthandler -m pytest tests/test_gpu_parity.py -x -q -k "c3 or managed or pinned or random" > gpurun_out/r02bz/sel.log 2>&1; echo "selection exit $?: $(tail -1 gpurun_out/r02bz/sel.log)"
timeout 2400 python -X faulthandler -m pytest tests -x -q -m gpu > gpurun_out/r02bz/gputests.log 2>&1; echo "suite exit $?: $(tail -1 gpurun_out/r02bz/gputests.log)"
for rep in 1 2; do
for m in 1 0; do
CRAC_HOST_NT=$m timeout 600 python bench.py --workload c3 --no-stall --no-cpu-baseline --no-verify > gpurun_out/r02bz/c3_nt${m}_$rep.json 2>gpurun_out/r02bz/c3_nt${m}_$rep.err
python -c "
import json; d=json.loads(open('gpurun_out/r02bz/c3_nt${m}_$rep.json').read().splitlines()[-1]); r=d['roofline']
print('c3 nt=$m', d['value'], d['e2e']['value'], d['per_gpu']['checkpoint_ms'], d['per_gpu']['restart_ms'], r['d2h_GBps_per_step'])"
done
done
