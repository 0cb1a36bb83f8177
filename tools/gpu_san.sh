#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_sanitizer.py -m gpu -q > gpurun_out/pytest_san.log 2>&1; echo "san rc=$?"; tail -5 gpurun_out/pytest_san.log
timeout 600 python bench.py --frames 2048 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C2_2048.json 2>/dev/null; cut -c1-300 gpurun_out/bench_C2_2048.json
