O=gpurun_out/r02/joint; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_joint.py -x -q -p no:cacheprovider 2>&1 | tail -3
for j in 4 8 3; do timeout 300 python bench.py --joint $j --frames 4096 > $O/bench_joint$j.json 2>$O/bench_joint$j.err; python -c "
import json; d=json.loads(open('$O/bench_joint$j.json').read()); print($j, round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"; done
