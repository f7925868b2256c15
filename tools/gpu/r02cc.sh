# round 2cc: every GPU test alone in a fresh process (first-drain-of-a-process bugs like the split-drain event read)
mkdir -p gpurun_out/r02cc
pass=0; fail=0
while read -r node; do
  [ -z "$node" ] && continue
  if timeout 300 python -X faulthandler -m pytest -x -q -p no:cacheprovider "$node" > gpurun_out/r02cc/last.log 2>&1; then
    pass=$((pass+1))
  else
    fail=$((fail+1)); echo "FAIL $node" >> gpurun_out/r02cc/failures.txt; tail -30 gpurun_out/r02cc/last.log >> gpurun_out/r02cc/failures.txt
  fi
done < tools/gpu/gpu_nodes_reversed.txt
echo "alone: $pass passed, $fail failed" | tee gpurun_out/r02cc/summary.txt
