# round 2an: split incremental drain: writer CTA count (C5, 64 GiB)
mkdir -p gpurun_out/r02an
for w in 16 24 32 8; do
CRAC_INCR_WRITERS=$w timeout 900 python bench.py --workload c5 --steps 3 --warmup 2 --no-stall --no-verify > gpurun_out/r02an/c5_$w.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/r02an/c5_$w.json').read().splitlines()[-1]); r=d['incremental']; print('writers=$w', {k: (v['drain_ms'], v['drain_roofline_ms'], v['hash_only_ms']) for k,v in r.items()})"
done
