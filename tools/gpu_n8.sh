#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for g in nccl p2p; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 2965$([ $g = nccl ] && echo 1 || echo 2) bench.py --gpus 8 --steps 5 --warmup 3 --dist-backend gloo --gather $g --no-e2e --scaling strong > gpurun_out/bench_n8_$g.json 2> gpurun_out/bench_n8_$g.err; echo "bench n8 $g rc=$?"; cut -c1-250 gpurun_out/bench_n8_$g.json; grep -iE "error|Traceback" gpurun_out/bench_n8_$g.err | head -5
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29655 tests/helpers/p2p_check.py --backend gloo > gpurun_out/p2p8.log 2>&1; echo "p2p8 rc=$?"; grep -c PASS gpurun_out/p2p8.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29656 tests/helpers/dist_check.py --backend gloo > gpurun_out/dist8.log 2>&1; echo "dist8 rc=$?"; grep PASS gpurun_out/dist8.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29657 bench.py --gpus 4 --impl reference --steps 2 --warmup 1 > gpurun_out/ref_n4.json 2> gpurun_out/ref_n4.err; echo "ref n4 rc=$?"; wc -l < gpurun_out/ref_n4.json
