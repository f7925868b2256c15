# round 2m: every bench workload on one B200 (tools/bench_all.sh), then the default bench line once more
OUT=gpurun_out/r02m bash tools/bench_all.sh > gpurun_out/r02m_all.log 2>&1; echo "all rc=$?"
tail -c 3000 gpurun_out/r02m_all.log
