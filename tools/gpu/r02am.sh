# round 2am: compute-sanitizer on every kernel path, final build
mkdir -p gpurun_out/r02am
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_paths.py > gpurun_out/r02am/sanitizer_$tool.txt 2>&1; echo "$tool rc=$?"
  tail -2 gpurun_out/r02am/sanitizer_$tool.txt
done
