# round 2ce: closing record of the exact last build: smoke, then every workload (bench_all)
mkdir -p gpurun_out/r02ce
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02ce/smoke.log 2>&1; tail -1 gpurun_out/r02ce/smoke.log
OUT=gpurun_out/r02ce/all bash tools/bench_all.sh > /dev/null 2>&1
for f in gpurun_out/r02ce/all/bench_*.json; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
except Exception as e:
    print(f, "unreadable", e); raise SystemExit
r = d.get("roofline") or {}; e = d.get("e2e") or {}; p = d.get("per_gpu") or {}; k = (r.get("kernels") or {}).get("k1_chunk_crc") or {}
inc = d.get("incremental") or {}; cpu = d.get("cpu_baseline") or {}
print(f.split("/")[-1], d.get("value"), e.get("value"), r.get("frac"), r.get("d2h_peak_GBps"), p.get("checkpoint_ms"), p.get("restart_ms"),
      "K1", k.get("frac"), "verified", (d.get("verified") or {}).get("ok"), "cpu", cpu.get("value"),
      {a: (b.get("drain_ms"), b.get("drain_roofline_ms")) for a, b in inc.items() if isinstance(b, dict) and "drain_ms" in b})
PY
done
