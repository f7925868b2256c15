# round 2o: full GPU suite + smoke after the pinned host hashing / cold full map / early-window rules
mkdir -p gpurun_out/r02o
timeout 1800 python -m pytest tests -q -m gpu --durations=12 > gpurun_out/r02o/gputests.log 2>&1; echo "tests rc=$?"
tail -22 gpurun_out/r02o/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02o/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02o/smoke.log
