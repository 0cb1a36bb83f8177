#!/bin/bash
# weak-scaling bench path with 2 and 4 ranks sharing one B200 (gloo process group), per-GPU
# share limited to 2,048 frames so the ranks fit one GPU's HBM; plus the strong split for comparison
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for n in 2 4; do
for sc in weak strong; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2967$n \
  bench.py --gpus $n --steps 5 --warmup 3 --dist-backend gloo --frames 2048 --scaling $sc --e2e-frames 64 \
  > gpurun_out/bench_n${n}_$sc.json 2> gpurun_out/bench_n${n}_$sc.err; echo "n$n $sc rc=$?"; cut -c1-420 gpurun_out/bench_n${n}_$sc.json
grep -iE "error|Traceback" gpurun_out/bench_n${n}_$sc.err | head -5
done
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29681 \
  bench.py --gpus 2 --impl reference --steps 2 --warmup 1 > gpurun_out/ref_n2.json 2> gpurun_out/ref_n2.err; echo "ref n2 rc=$?"; cut -c1-300 gpurun_out/ref_n2.json
