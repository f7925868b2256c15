# round 2ch: validation of the round's last build: full GPU suite, smoke, default bench, reference arm
mkdir -p gpurun_out/r02ch
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r02ch/gputests.log 2>&1; tail -1 gpurun_out/r02ch/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02ch/smoke.log 2>&1; tail -1 gpurun_out/r02ch/smoke.log
timeout 900 python bench.py > gpurun_out/r02ch/bench_c4.json 2> gpurun_out/r02ch/bench_c4.err
timeout 900 python bench.py --impl reference > gpurun_out/r02ch/bench_reference.json 2> gpurun_out/r02ch/bench_reference.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02ch/bench_c4.json").read().splitlines()[-1])
r = d["roofline"]; e = d["e2e"]
print("c4", d["value"], e["value"], e["with_teardown"]["value"], r["frac"], d["per_gpu"]["checkpoint_ms"], d["per_gpu"]["restart_ms"],
      r["d2h_peak_GBps"], "K1", r["kernels"]["k1_chunk_crc"]["frac"], "verified", d["verified"]["ok"], d["clocks"]["reasons"])
ref = json.loads(open("gpurun_out/r02ch/bench_reference.json").read().splitlines()[-1])
print("reference", ref.get("value"))
PY
