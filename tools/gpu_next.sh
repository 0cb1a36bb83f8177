#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_next.py -m gpu -q -x > gpurun_out/pytest_next.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_next.log
timeout 600 python bench.py --config C2 --cuts 16 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C2_cuts.json 2> gpurun_out/bench_C2_cuts.err; echo "C2cuts rc=$?"; cut -c1-300 gpurun_out/bench_C2_cuts.json; tail -3 gpurun_out/bench_C2_cuts.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621 bench.py --gpus 2 --cuts 16 --steps 3 --warmup 3 --dist-backend gloo --no-e2e --frames 2048 > gpurun_out/bench_n2_cuts.json 2> gpurun_out/bench_n2_cuts.err; echo "n2 cuts rc=$?"; cut -c1-300 gpurun_out/bench_n2_cuts.json; tail -3 gpurun_out/bench_n2_cuts.err
