# round 2br: the driver's round-end sequence on the final build: smoke, default bench, reference arm
mkdir -p gpurun_out/r02br
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02br/smoke.log 2>&1; tail -1 gpurun_out/r02br/smoke.log
timeout 900 python bench.py > gpurun_out/r02br/bench.json 2> gpurun_out/r02br/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r02br/bench_reference.json 2> gpurun_out/r02br/bench_reference.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02br/bench.json").read().splitlines()[-1])
r = d["roofline"]; e = d["e2e"]
print("bench", d["value"], e["value"], e["with_teardown"]["value"], r["frac"], d["per_gpu"]["checkpoint_ms"], d["per_gpu"]["restart_ms"],
      r["d2h_peak_GBps"], r["h2d_peak_GBps"], "K1", r["kernels"]["k1_chunk_crc"]["frac"], "verified", d["verified"]["ok"], "launches", d["gpu_launches"], d["clocks"])
ref = json.loads(open("gpurun_out/r02br/bench_reference.json").read().splitlines()[-1])
print("reference", ref.get("value"), ref.get("cpu_baseline", {}).get("cores"), "ratio e2e", round(e["value"] / ref["value"], 2))
PY
