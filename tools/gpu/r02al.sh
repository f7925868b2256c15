# round 2al: launch list of the final build (bench command at 96 GiB: 120 GiB is OOM-killed under ncu on this host)
NCU=/usr/local/cuda/bin/ncu
OUT=gpurun_out/r02q2
mkdir -p $OUT
timeout 3000 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv \
  --log-file $OUT/launches.csv python bench.py --footprint-gib 96 --steps 1 --warmup 1 \
  --no-cpu-baseline --no-incremental --no-stall --no-verify > $OUT/launches_bench.log 2>&1
echo "launch run exit $?"
