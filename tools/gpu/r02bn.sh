# round 2bn: every workload on the final build (bench_all), recorded with the box's link peaks
mkdir -p gpurun_out/r02bn
OUT=gpurun_out/r02bn/all bash tools/bench_all.sh > /dev/null 2>&1
for f in gpurun_out/r02bn/all/bench_*.json; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
except Exception as e:
    print(f, "unreadable", e); raise SystemExit
r = d.get("roofline") or {}; e = d.get("e2e") or {}; p = d.get("per_gpu") or {}; k = (r.get("kernels") or {}).get("k1_chunk_crc") or {}
inc = d.get("incremental") or {}; cpu = d.get("cpu_baseline") or {}
print(f.split("/")[-1], d.get("value"), e.get("value"), (e.get("with_teardown") or {}).get("value"), r.get("frac"),
      r.get("d2h_peak_GBps"), r.get("h2d_peak_GBps"), p.get("checkpoint_ms"), p.get("restart_ms"), "K1", k.get("frac"),
      "verified", (d.get("verified") or {}).get("ok"), "cpu", cpu.get("value"),
      {a: (b.get("drain_ms"), b.get("drain_roofline_ms"), b.get("hash_frac_of_hbm")) for a, b in inc.items() if isinstance(b, dict) and "drain_ms" in b})
PY
done
