#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_shapes or content" > gpurun_out/pytest_b256.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_b256.log
for r in 1 2; do timeout 600 python bench.py --bins 256 --no-cpu-baseline --no-e2e > gpurun_out/bench_b256_$r.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_b256_$r.json')); r=d['roofline']; print('bins256 film', round(d['value']), round(r['achieved']), round(r['frac'],3), d['clocks']['reasons'])"; done
timeout 600 python bench.py --bins 256 --frames 4096 --no-cpu-baseline --no-e2e > gpurun_out/bench_b256_4096.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_b256_4096.json')); r=d['roofline']; print('bins256 4096f', round(d['value']), round(r['achieved']), round(r['frac'],3))"
