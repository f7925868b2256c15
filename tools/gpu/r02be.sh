# round 2be: final validation of the round-2 build (direct D2H drain, K1 on 144 SMs, streamed file write, e2e
# through the two API calls): full GPU suite, smoke, every workload, then the launch list of the bench command
# and ncu full sets of the drain's K1 and its edge pack.  Outputs gpurun_out/r02be.
mkdir -p gpurun_out/r02be
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r02be/gputests.log 2>&1; tail -3 gpurun_out/r02be/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02be/smoke.log 2>&1; tail -1 gpurun_out/r02be/smoke.log
OUT=gpurun_out/r02be/all bash tools/bench_all.sh > /dev/null 2>&1
for f in gpurun_out/r02be/all/bench_*.json; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
except Exception as e:
    print(f, "unreadable", e); raise SystemExit
r = d.get("roofline") or {}; e = d.get("e2e") or {}; cpu = d.get("cpu_baseline") or {}; p = d.get("per_gpu") or {}
print(f.split("/")[-1], d.get("value"), e.get("value"), (e.get("with_teardown") or {}).get("value"), r.get("frac"),
      p.get("checkpoint_ms"), p.get("restart_ms"), "verified", (d.get("verified") or {}).get("ok"), "cpu", cpu.get("value"), cpu.get("kind"))
PY
done
NCU=/usr/local/cuda/bin/ncu
OUT=gpurun_out/r02be/ncu
mkdir -p $OUT
BENCH8="python bench.py --footprint-gib 8 --steps 1 --warmup 1 --no-cpu-baseline --no-incremental --no-stall --no-verify --no-cold"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k1_chunk_crc -s 5 -c 1 \
  -o $OUT/prof_k1_drain $BENCH8 > $OUT/prof_k1_drain.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_pack_records -s 200 -c 1 \
  -o $OUT/prof_k_pack_records $BENCH8 > $OUT/prof_k_pack_records.log 2>&1
timeout 3000 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv \
  --log-file $OUT/launches.csv python bench.py --footprint-gib 96 --steps 1 --warmup 1 \
  --no-cpu-baseline --no-incremental --no-stall --no-verify --no-cold > $OUT/launches_bench.log 2>&1
echo "launch run exit $?" >> $OUT/launches_bench.log
ls -la $OUT
