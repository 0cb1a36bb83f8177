#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py -m gpu -q -x -k "fused or torchrun or local_dest" > gpurun_out/pytest_p2p.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_p2p.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --gather p2p --no-e2e --frames 4096 > gpurun_out/bench_n2_p2p.json 2> gpurun_out/bench_n2_p2p.err; echo "bench p2p rc=$?"; cut -c1-400 gpurun_out/bench_n2_p2p.json; tail -5 gpurun_out/bench_n2_p2p.err
