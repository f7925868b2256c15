# round 2cb: order-dependence hunt -- the GPU tests in reverse order, in a seeded shuffle, and each file in its own process
mkdir -p gpurun_out/r02cb
timeout 1500 python -X faulthandler -m pytest -x -q -p no:cacheprovider $(cat tools/gpu/gpu_nodes_reversed.txt) > gpurun_out/r02cb/reversed.log 2>&1; echo "reversed exit $?: $(tail -1 gpurun_out/r02cb/reversed.log)"
timeout 1500 python -X faulthandler -m pytest -x -q -p no:cacheprovider $(cat tools/gpu/gpu_nodes_shuffled7.txt) > gpurun_out/r02cb/shuffled7.log 2>&1; echo "shuffled exit $?: $(tail -1 gpurun_out/r02cb/shuffled7.log)"
for f in tests/test_gpu_*.py; do
timeout 900 python -X faulthandler -m pytest -x -q -p no:cacheprovider $f > gpurun_out/r02cb/$(basename $f .py).log 2>&1; echo "$f exit $?: $(tail -1 gpurun_out/r02cb/$(basename $f .py).log)"
done
