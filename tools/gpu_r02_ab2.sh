#!/bin/bash
# same-box A/B: the library before this session's kVarGen changes (old) vs HEAD (new)
O=${OUT:-gpurun_out/r02/ab2}; mkdir -p $O
P=paper_1805_07339_b200
make -j8 all > $O/make.log 2>&1 || { tail $O/make.log; exit 1; }
cp $P/libscn.so $P/libscn_ab_new.so
T="python tools/hist_tune.py shots"
for r in 1 2 3; do for v in ${AB_LIBS:-old new}; do
  cp $P/libscn_ab_$v.so $P/libscn.so
  for sh in 1366x768 854x480 426x240; do for op in histds ds; do
    $T 2048 C4 $op --shape $sh | sed "s/^{/{\"ab\": \"$v\", /" >> $O/tune.jsonl
  done; done
  $T 1024 C4 ds --offset 4 | sed "s/^{/{\"ab\": \"$v\", /" >> $O/tune.jsonl
done; done
cp $P/libscn_ab_new.so $P/libscn.so
python - <<'PY'
import json,os,collections
r=collections.defaultdict(list)
for l in open(os.environ.get("OUT","gpurun_out/r02/ab2")+"/tune.jsonl"):
    d=json.loads(l); r[(d['op'],d['width'],d['offset'],d['ab'])].append(round(d['GBps']))
for k,v in sorted(r.items()): print(k, v)
PY
[ -n "$NO_PROF" ] && exit 0
# source-level capture of the current fused realigning kernel (1366x768)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hist_tma_kernel -s 3 -c 1 -o $O/full_histds_1366 \
  python tools/hist_tune.py shots 512 C4 histds --shape 1366x768 --reps 1 > $O/full_histds_1366.log 2>&1; echo "ncu $?"
ncu -i $O/full_histds_1366.ncu-rep --page source --csv --print-source sass > $O/src_sass.csv 2>&1; echo "src $?"
rm -f $O/full_histds_1366.ncu-rep
