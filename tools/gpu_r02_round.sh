#!/bin/bash
# r02 round pass on one B200: tests, smoke, every bench line, reference arm, ncu evidence.
# Everything lands in gpurun_out/r02/round/ (copied to profiles/ by hand).
O=${ROUND_OUT:-gpurun_out/r02/round}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit,driver_version --format=csv > $O/box.txt
nproc >> $O/box.txt; lscpu | grep "Model name" >> $O/box.txt
if [ "${1:-}" != "notest" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -3 $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
fi
# traffic summaries of THIS library first, so every bench line's roofline.traffic_source matches it
bash tools/gpu_r02_traffic.sh > $O/traffic_pass.log 2>&1; cp gpurun_out/r02/traffic/ncu_*_summary.json profiles/; echo "traffic $?"
B="timeout 900 python bench.py"
$B > $O/bench_C2.json 2> $O/bench_C2.err; echo "C2 $?"
$B --frames 2048 --no-cpu-baseline --no-e2e > $O/bench_C2_2048f_shard_proxy.json 2>/dev/null; echo "proxy $?"
$B --config C3 --cpu-seconds 5 > $O/bench_C3.json 2>/dev/null; echo "C3 $?"
$B --config C4 --cpu-seconds 5 > $O/bench_C4.json 2>/dev/null; echo "C4 $?"
$B --config C5 --frames 4096 --steps 10 --cpu-seconds 5 --e2e-frames 64 > $O/bench_C5.json 2>/dev/null; echo "C5 $?"
$B --config C5 --round-frames 3584 --steps 5 --warmup 3 > $O/bench_C5_rounds.json 2>/dev/null; echo "C5 rounds $?"
$B --bins 100 --no-cpu-baseline --no-e2e > $O/bench_C2_bins100.json 2>/dev/null; echo "b100 $?"
$B --bins 256 --no-cpu-baseline --no-e2e > $O/bench_C2_bins256.json 2>/dev/null; echo "b256 $?"
$B --bins 100 --frames 4096 --no-cpu-baseline --no-e2e > $O/bench_C2_bins100_4096f.json 2>/dev/null; echo "b100 4096 $?"
$B --config C4 --shape 1366x768 --no-cpu-baseline --no-e2e > $O/bench_C4_1366x768.json 2>/dev/null; echo "1366 $?"
$B --config C4 --shape 854x480 --no-cpu-baseline --no-e2e > $O/bench_C4_854x480.json 2>/dev/null; echo "854 $?"
$B --config C3 --graph e > $O/bench_C3_graph_e.json 2>/dev/null; echo "C3e $?"
$B --cuts 16 --no-cpu-baseline --no-e2e > $O/bench_C2_cuts16.json 2>/dev/null; echo "cuts $?"
$B --montage 8 --steps 10 > $O/bench_C2_montage8.json 2>/dev/null; echo "montage $?"
for m in uniform constant xgrad; do $B --mode $m --no-cpu-baseline --no-e2e > $O/bench_C2_$m.json 2>/dev/null; echo "$m $?"; done
for impl in 1 2; do $B --hist-impl $impl --frames 1024 --steps 5 --no-cpu-baseline --no-e2e > $O/bench_C2_k2a_impl$impl.json 2>/dev/null; echo "k2a $impl $?"; done
for g in nccl p2p; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=$((20000 + RANDOM % 20000)) bench.py --gpus 2 --dist-backend gloo --gather $g --no-e2e --no-cpu-baseline --steps 10 > $O/bench_n2_shared_gpu_$g.json 2>$O/bench_n2_shared_gpu_$g.err; echo "n2 $g $?"; done
for j in 8 4 3; do $B --joint $j > $O/bench_C2_joint$j.json 2>/dev/null; echo "joint $j $?"; done
$B --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>/dev/null; echo "ref $?"
NCU_OUT=$O/ncu bash tools/gpu_r02_ncu.sh > $O/ncu_pass.log 2>&1; echo "ncu $?"
T="python tools/hist_tune.py shots"
for r in 1 2; do for sh in 1366x768 854x480 426x240; do for op in histds ds; do $T 2048 C4 $op --shape $sh >> $O/tune_gen.jsonl 2>/dev/null; done; done; done
