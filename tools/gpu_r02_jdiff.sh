#!/bin/bash
# joint-colour shot-diff: GPU parity + bench lines; C2 sanity line
O=gpurun_out/r02/jdiff; mkdir -p $O
make -j8 all > $O/make.log 2>&1 || { tail $O/make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_joint.py -q -p no:cacheprovider > $O/pytest_joint.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_joint.log
B="timeout 600 python bench.py"
for j in 8 4 3; do $B --joint $j > $O/bench_C2_joint$j.json 2>$O/joint$j.err; echo "joint $j $?"; done
$B --no-cpu-baseline --no-e2e > $O/bench_C2.json 2>$O/c2.err; echo "C2 $?"
cat $O/*.json | python -c "import sys,json;[print(round(d['value']),d['roofline']['achieved'],d['config'].get('ops'),d['clocks']['sm_mhz']) for d in map(json.loads,sys.stdin)]"
