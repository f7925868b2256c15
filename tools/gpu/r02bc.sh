# round 2bc: e2e without the teardown (with_teardown beside it), K1 with 4 spare SMs: C4, C3, C2
mkdir -p gpurun_out/r02bc
timeout 900 python bench.py > gpurun_out/r02bc/bench_c4.json 2> gpurun_out/r02bc/bench_c4.err
timeout 600 python bench.py --workload c3 > gpurun_out/r02bc/bench_c3.json 2> gpurun_out/r02bc/bench_c3.err
timeout 600 python bench.py --workload c2 > gpurun_out/r02bc/bench_c2.json 2> gpurun_out/r02bc/bench_c2.err
for w in c4 c3 c2; do python - gpurun_out/r02bc/bench_$w.json <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
except Exception as e:
    print(f, "unreadable", e); raise SystemExit
r = d.get("roofline") or {}; e = d.get("e2e") or {}; k = r.get("kernels") or {}
print(f.split("/")[-1], d.get("value"), e.get("value"), (e.get("with_teardown") or {}).get("value"), r.get("frac"),
      (d.get("per_gpu") or {}).get("checkpoint_ms"), (d.get("per_gpu") or {}).get("restart_ms"),
      e.get("api_ms_per_step"), e.get("teardown_ms_per_step"), "K1", (k.get("k1_chunk_crc") or {}).get("frac"),
      "verified", (d.get("verified") or {}).get("ok"))
PY
done
