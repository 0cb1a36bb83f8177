#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_multirank.py -m gpu -q > gpurun_out/pytest_mr.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_mr.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --no-e2e --frames 4096 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "bench n2 rc=$?"; cut -c1-300 gpurun_out/bench_n2.json
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['gpu_launches'], d['roofline']['kernel'])"
