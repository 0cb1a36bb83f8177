O=gpurun_out/r02/ncu2
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hist_tma_kernel -s 3 -c 1 -o $O/full_histds_1366 \
  python tools/hist_tune.py shots 512 C4 histds --shape 1366x768 --reps 1 > $O/full_histds_1366.log 2>&1; echo "gen histds $?"
for g in nccl p2p; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=$((20000 + RANDOM % 20000)) bench.py --gpus 2 --dist-backend gloo --gather $g --no-e2e --no-cpu-baseline --steps 10 > $O/bench_n2_shared_gpu_$g.json 2>$O/bench_n2_shared_gpu_$g.err; echo "n2 $g $?"; tail -c 300 $O/bench_n2_shared_gpu_$g.err; done
