#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_next.py -m gpu -q -x > gpurun_out/pytest_next.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_next.log
timeout 600 python bench.py --config C2 --montage 8 --steps 5 --warmup 2 > gpurun_out/bench_C2_montage.json 2> gpurun_out/bench_C2_montage.err; echo "montage rc=$?"; cut -c1-600 gpurun_out/bench_C2_montage.json; tail -3 gpurun_out/bench_C2_montage.err
