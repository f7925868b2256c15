# round 2bf: the final build's bench lines again on another box (r02be's box had a 39.5 GB/s D2H link): C4 x2, C2, C5, C3
mkdir -p gpurun_out/r02bf
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02bf/gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02bf/bench_c4.json 2> gpurun_out/r02bf/bench_c4.err
timeout 900 python bench.py > gpurun_out/r02bf/bench_c4_2.json 2> gpurun_out/r02bf/bench_c4_2.err
timeout 600 python bench.py --workload c2 > gpurun_out/r02bf/bench_c2.json 2> gpurun_out/r02bf/bench_c2.err
timeout 600 python bench.py --workload c3 > gpurun_out/r02bf/bench_c3.json 2> gpurun_out/r02bf/bench_c3.err
timeout 900 python bench.py --workload c5 > gpurun_out/r02bf/bench_c5.json 2> gpurun_out/r02bf/bench_c5.err
for f in gpurun_out/r02bf/bench_*.json; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
except Exception as e:
    print(f, "unreadable", e); raise SystemExit
r = d.get("roofline") or {}; e = d.get("e2e") or {}; p = d.get("per_gpu") or {}; k = (r.get("kernels") or {}).get("k1_chunk_crc") or {}
inc = d.get("incremental") or {}
print(f.split("/")[-1], d.get("value"), e.get("value"), (e.get("with_teardown") or {}).get("value"), r.get("frac"),
      r.get("d2h_peak_GBps"), r.get("h2d_peak_GBps"), p.get("checkpoint_ms"), p.get("restart_ms"), "K1", k.get("frac"),
      "verified", (d.get("verified") or {}).get("ok"),
      {a: (b.get("drain_ms"), b.get("drain_roofline_ms"), b.get("hash_frac_of_hbm")) for a, b in inc.items() if isinstance(b, dict) and "drain_ms" in b})
PY
done
