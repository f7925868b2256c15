# round 2bw: reproduce r02bv's segfault in test_async_drain_with_managed_runs_matches_reference (NT host copy on / off)
mkdir -p gpurun_out/r02bw
for rep in 1 2 3; do
for m in 1 0; do
CRAC_HOST_NT=$m timeout 300 python -X faulthandler -m pytest tests/test_gpu_parity.py -x -q -k "async_drain_with_managed_runs or async_drain_is_the_image" > gpurun_out/r02bw/t_nt${m}_$rep.log 2>&1
echo "nt=$m rep=$rep exit $?: $(tail -1 gpurun_out/r02bw/t_nt${m}_$rep.log)"
done
done
