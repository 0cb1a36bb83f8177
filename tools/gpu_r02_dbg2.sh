make tuning > /dev/null 2>&1
export SCN_LIB=tuning
for g in 7 1; do
for args in "854 480 3 hist" "854 480 3 ds" "854 480 3 fused" "960 64 3 fused" "960 64 3 ds" "67 41 20 fused" "67 41 20 ds" "64 36 20 fused"; do
  echo "== GRID=$g $args"; SCN_GRID=$g timeout 30 python tools/dbg_gen.py $args 2>&1 | tail -2
done
done
