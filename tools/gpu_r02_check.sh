#!/bin/bash
# full GPU suite + smoke + the realigning bench lines on the current library
O=${OUT:-gpurun_out/r02/check}; mkdir -p $O
make -j8 all > $O/make.log 2>&1 || { tail $O/make.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
B="timeout 900 python bench.py"
$B --config C4 --shape 1366x768 --no-cpu-baseline --no-e2e > $O/bench_C4_1366x768.json 2>/dev/null; echo "1366 $?"
$B --config C4 --shape 854x480 --no-cpu-baseline --no-e2e > $O/bench_C4_854x480.json 2>/dev/null; echo "854 $?"
$B --no-cpu-baseline --no-e2e > $O/bench_C2.json 2>/dev/null; echo "C2 $?"
for f in $O/bench_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"; done
