mkdir -p gpurun_out/r02
for args in "1366 768 3 ds" "1366 768 3 fused" "854 480 3 fused"; do
  echo "== $args"; timeout 60 python tools/dbg_gen.py $args 2>&1 | tail -3
done
timeout 600 python -m pytest tests/test_gpu_gen.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=30 > gpurun_out/r02/pytest_gpu_t2.log 2>&1
echo "pytest rc=$?"
tail -45 gpurun_out/r02/pytest_gpu_t2.log
