# round 2e: barrier + parity GPU tests after the arena-cache fix, verify API; ncu of K1 with / without the key lane
mkdir -p gpurun_out/r02e
timeout 900 python -m pytest tests/test_gpu_barrier.py tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q > gpurun_out/r02e/gputests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r02e/gputests.log
for c in 16:nokey 8:key; do
  n=$(echo $c | tr ':' '_')
  timeout 600 ncu --set full --clock-control none -k regex:k1_chunk_crc -s 2 -c 1 -o gpurun_out/r02e/k1_$n python tools/exp_k1_key.py $c > gpurun_out/r02e/ncu_$n.log 2>&1; echo "ncu $c rc=$?"
done
