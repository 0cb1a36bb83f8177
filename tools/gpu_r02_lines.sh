#!/bin/bash
# re-take the bench lines whose roofline.traffic comes from a profiles/ncu_*_summary.json capture
O=${OUT:-gpurun_out/r02/lines}; mkdir -p $O
B="timeout 900 python bench.py"
$B > $O/bench_C2.json 2> $O/bench_C2.err; echo "C2 $?"
$B --frames 2048 --no-cpu-baseline --no-e2e > $O/bench_C2_2048f_shard_proxy.json 2>/dev/null; echo "proxy $?"
$B --config C3 --cpu-seconds 5 > $O/bench_C3.json 2>/dev/null; echo "C3 $?"
$B --config C4 --cpu-seconds 5 > $O/bench_C4.json 2>/dev/null; echo "C4 $?"
$B --config C5 --frames 4096 --steps 10 --cpu-seconds 5 --e2e-frames 64 > $O/bench_C5.json 2>/dev/null; echo "C5 $?"
for f in $O/bench_*.json; do python -c "import json; d=json.load(open('$f')); r=d['roofline']; print('$f', round(d['value']), round(r['achieved']), r.get('traffic_source',{}).get('matches_library'), d['clocks']['sm_mhz'])"; done
