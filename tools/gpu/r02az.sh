# round 2az: direct D2H drain by default: full GPU suite, smoke, every workload
mkdir -p gpurun_out/r02az
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r02az/gputests.log 2>&1; tail -3 gpurun_out/r02az/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02az/smoke.log 2>&1; tail -1 gpurun_out/r02az/smoke.log
OUT=gpurun_out/r02az/all bash tools/bench_all.sh > /dev/null 2>&1
for f in gpurun_out/r02az/all/bench_*.json; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
except Exception as e:
    print(f, "unreadable", e); raise SystemExit
r = d.get("roofline") or {}
cpu = d.get("cpu_baseline") or {}
k = (r.get("kernels") or {}).get("k_pack_records") or {}
print(f.split("/")[-1], d.get("value"), (d.get("e2e") or {}).get("value"), r.get("frac"),
      (d.get("per_gpu") or {}).get("checkpoint_ms"), (d.get("per_gpu") or {}).get("restart_ms"),
      "pack", k.get("launches"), k.get("avg_launch_ms"), "cpu", cpu.get("value"))
PY
done
