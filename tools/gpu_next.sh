#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_shapes or content" > gpurun_out/pytest_n4.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_n4.log
for b in 256 64 32 100 17; do timeout 600 python bench.py --config C2 --bins $b --frames 4096 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C2_b$b.json 2> gpurun_out/bench_C2_b$b.err; echo "bins $b rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_C2_b$b.json')); r=d['roofline']; print($b, round(d['value']), round(r['achieved']), round(r['frac'],3), d['config']['hist_variant'])"; done
for m in uniform constant; do timeout 600 python bench.py --config C2 --bins 256 --mode $m --frames 4096 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C2_b256_$m.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_C2_b256_$m.json')); r=d['roofline']; print('256 $m', round(d['value']), round(r['achieved']), round(r['frac'],3))"; done
