mkdir -p gpurun_out/r02
for args in "1366 768 3 hist" "1366 768 3 ds" "1366 768 3 fused" "1366 100 3 fused" "1366 200 1 fused" "854 480 3 fused" "1366 768 1 ds"; do
  echo "== $args"; timeout 60 python tools/dbg_gen.py $args 2>&1 | tail -5; echo "rc=$?"
done
timeout 300 compute-sanitizer --tool memcheck python tools/dbg_gen.py 1366 100 1 fused 2>&1 | tail -20
