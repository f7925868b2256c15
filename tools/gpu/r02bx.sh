# round 2bx: r02bv's test selection again (its run segfaulted in test_async_drain_with_managed_runs after 13 tests), NT on / off
mkdir -p gpurun_out/r02bx
for rep in 1 2; do
for m in 1 0; do
CRAC_HOST_NT=$m timeout 600 python -X faulthandler -m pytest tests/test_gpu_parity.py -x -q -k "c3 or managed or pinned or random" > gpurun_out/r02bx/t_nt${m}_$rep.log 2>&1
echo "nt=$m rep=$rep exit $?: $(tail -1 gpurun_out/r02bx/t_nt${m}_$rep.log | cut -c1-200)"
done
done
