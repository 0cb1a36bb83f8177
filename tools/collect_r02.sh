#!/bin/bash
# copy a round pass (tools/gpu_r02_round.sh output dir) into profiles/ under the r02_ names
set -e
S=${1:-gpurun_out/r02/final2}
P=profiles
for f in $S/bench_*.json; do b=$(basename $f .json); cp $f $P/r02_${b}.json; done
for f in $S/ncu/counters_*.json; do b=$(basename $f .json); cp $f $P/r02_ncu_${b}.json; done
for f in $S/ncu/ncu_*_summary.json; do cp $f $P/; done
cp $S/ncu/launches_bench.csv $P/r02_launches_C2_4096f.csv
cp $S/pytest_gpu.log $P/r02_pytest_gpu.log
cp $S/smoke.log $P/r02_smoke.log
cp $S/box.txt $P/r02_box_info.txt
python - "$S" <<'PY'
import json, sys
S = sys.argv[1]
with open("profiles/r02_tune_gen.jsonl", "a") as out:
    for l in open(S + "/tune_gen.jsonl"):
        d = json.loads(l); d["experiment"] = "final round pass " + S; out.write(json.dumps(d) + "\n")
PY
ls $S/ncu/*summary.json
