# r02 bench lines (N = 1 unless stated) after the library strip + kVarGen kernels
mkdir -p gpurun_out/r02/bench
O=gpurun_out/r02/bench
B="timeout 900 python bench.py"
$B > $O/c2_default.json 2> $O/c2_default.err; echo "c2 default $?"
$B --frames 2048 --no-cpu-baseline --no-e2e > $O/c2_2048.json 2>/dev/null; echo "c2 2048 $?"
$B --frames 2048 --no-cpu-baseline --no-e2e --no-graph > $O/c2_2048_eager.json 2>/dev/null; echo "c2 2048 eager $?"
$B --bins 100 --no-cpu-baseline --no-e2e > $O/c2_b100.json 2>/dev/null; echo "b100 $?"
$B --bins 256 --no-cpu-baseline --no-e2e > $O/c2_b256.json 2>/dev/null; echo "b256 $?"
$B --config C4 --no-cpu-baseline --no-e2e > $O/c4.json 2>/dev/null; echo "c4 $?"
$B --config C4 --shape 1366x768 --no-cpu-baseline --no-e2e > $O/c4_1366.json 2>/dev/null; echo "c4 1366 $?"
$B --config C4 --shape 854x480 --no-cpu-baseline --no-e2e > $O/c4_854.json 2>/dev/null; echo "c4 854 $?"
$B --config C4 --shape 426x240 --no-cpu-baseline --no-e2e > $O/c4_426.json 2>/dev/null; echo "c4 426 $?"
$B --config C3 --no-cpu-baseline --no-e2e > $O/c3.json 2>/dev/null; echo "c3 $?"
for sh in 1366x768 854x480; do
  for op in ds histds; do python tools/hist_tune.py shots 2048 C4 $op --shape $sh >> $O/tune_gen.jsonl 2>/dev/null; done
  python tools/hist_tune.py shots 2048 C4 ds --shape $sh --offset 3 >> $O/tune_gen.jsonl 2>/dev/null
done
for op in ds histds; do python tools/hist_tune.py shots 1024 C4 $op >> $O/tune_gen.jsonl 2>/dev/null; python tools/hist_tune.py shots 1024 C4 $op --offset 4 >> $O/tune_gen.jsonl 2>/dev/null; done
for impl in 1 2; do python tools/hist_tune.py shots 256 C2 hist --impl $impl >> $O/tune_k2a.jsonl 2>/dev/null; python tools/hist_tune.py uniform 256 C2 hist --impl $impl >> $O/tune_k2a.jsonl 2>/dev/null; python tools/hist_tune.py constant 256 C2 hist --impl $impl >> $O/tune_k2a.jsonl 2>/dev/null; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29533 bench.py --gpus 2 --dist-backend gloo --no-e2e --no-cpu-baseline --steps 10 > $O/n2_gloo.json 2>$O/n2_gloo.err; echo "n2 gloo $?"
$B --impl reference --steps 3 --warmup 3 > $O/ref.json 2>/dev/null; echo "ref $?"
for f in $O/*.json; do python - "$f" <<'PY'
import json,sys
f=sys.argv[1]
try:
    d=json.loads(open(f).read().strip().splitlines()[-1])
except Exception as e:
    print(f, "ERR", e); sys.exit()
r=d.get("roofline") or {}
print(f.split("/")[-1], round(d["value"]), round(d["ms_per_step"],3), round(r.get("achieved") or 0), d.get("breakdown",{}).get("overhead_ms"), (d.get("e2e") or {}).get("value"), d.get("config",{}).get("step_launch"))
PY
done
cat $O/tune_gen.jsonl $O/tune_k2a.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['op'], d['width'], d['offset'], d['mode'], d['impl'], round(d['GBps']), d['variant'])"
