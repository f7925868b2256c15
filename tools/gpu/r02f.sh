# round 2f: full GPU suite (barrier, verify, arena cache fix), smoke, C4 bench with the new accounting, ncu K1 key/nokey
mkdir -p gpurun_out/r02f
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r02f/gputests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r02f/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02f/smoke.log
for c in 16:nokey 8:key; do
  n=$(echo $c | tr ':' '_')
  timeout 600 ncu --set full --clock-control none -k regex:k1_chunk_crc -s 2 -c 1 -o gpurun_out/r02f/k1_$n python tools/exp_k1_key.py $c > gpurun_out/r02f/ncu_$n.log 2>&1; echo "ncu $c rc=$?"
done
timeout 900 python bench.py --steps 3 --warmup 3 --no-stall > gpurun_out/r02f/bench_c4.json 2> gpurun_out/r02f/bench_c4.err; echo "c4 rc=$?"
tail -3 gpurun_out/r02f/bench_c4.err
