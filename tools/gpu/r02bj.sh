# round 2bj: full GPU suite + smoke on the build with the batched small-stream verify and the drain threads' device binding
mkdir -p gpurun_out/r02bj
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r02bj/gputests.log 2>&1; tail -3 gpurun_out/r02bj/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02bj/smoke.log 2>&1; tail -1 gpurun_out/r02bj/smoke.log
