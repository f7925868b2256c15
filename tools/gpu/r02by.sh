# round 2by: narrow the async-drain segfault: the pinned all-shadow test then the managed async test, with a C backtrace
mkdir -p gpurun_out/r02by
which gdb > gpurun_out/r02by/gdb.txt 2>&1
A="tests/test_gpu_parity.py::test_pinned_payloads_move_on_the_host_and_match_reference[all-shadow]"
B="tests/test_gpu_parity.py::test_async_drain_with_managed_runs_matches_reference[64]"
C="tests/test_gpu_parity.py::test_pinned_payloads_move_on_the_host_and_match_reference[ring+shadow]"
timeout 300 python -X faulthandler -m pytest -x -q "$A" "$B" > gpurun_out/r02by/ab.log 2>&1; echo "A,B exit $?"
timeout 300 python -X faulthandler -m pytest -x -q "$C" "$B" > gpurun_out/r02by/cb.log 2>&1; echo "C,B exit $?"
if [ -s gpurun_out/r02by/gdb.txt ] && grep -q gdb gpurun_out/r02by/gdb.txt; then
  CRAC_TRACE=1 timeout 600 gdb -batch -ex run -ex bt -ex "thread apply all bt 8" --args python -m pytest -x -q "$A" "$B" > gpurun_out/r02by/gdb_bt.log 2>&1
  echo "gdb exit $?"
else
  CRAC_TRACE=1 timeout 300 python -X faulthandler -m pytest -x -q "$A" "$B" > gpurun_out/r02by/trace.log 2>&1; echo "trace exit $?"
fi
