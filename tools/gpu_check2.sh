#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_sanitizer.py -m gpu -q > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?"; tail -40 gpurun_out/pytest_gpu2.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --no-e2e > gpurun_out/bench_n2_gloo.json 2> gpurun_out/bench_n2_gloo.err; echo "bench n2 rc=$?"; cat gpurun_out/bench_n2_gloo.json; tail -5 gpurun_out/bench_n2_gloo.err
