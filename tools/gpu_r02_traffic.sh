# re-capture the ncu traffic summaries bench.py reads (roofline.traffic) for the current library
O=gpurun_out/r02/traffic; mkdir -p $O
SHA=$(python -c "import paper_1805_07339_b200 as s; print(s.scn_version().split(', ')[1].rstrip(')'))")
cap() {  # name cfg frames op F desc
  timeout 900 ncu --set full --clock-control none -k regex:hist_tma_kernel -s 3 -c 1 -o $O/full_$1 \
    python tools/hist_tune.py shots $3 $2 $4 --reps 1 > $O/full_$1.log 2>&1
  python tools/ncu_traffic.py $O/full_$1.ncu-rep $4 $3 $5 $SHA $O/ncu_$1_summary.json "$6"
}
cap hist C2 2048 hist 6220800 "hist_tma_kernel<0,16>, C2 shape, 2048 frames/launch"
cap histds C4 1024 histds 6220800 "hist_tma_kernel<2,8> fused hist+downsample, C4 shape, 1024 frames/launch"
cap hist_c3 C3 8192 hist 691200 "hist_tma_kernel<0,16>, C3 shape 640x360, 8192 frames/launch"
cap histds_4k C5 512 histds 24883200 "hist_tma_kernel<2,8> fused hist+downsample, C5 shape 3840x2160, 512 frames/launch"
python bench.py --frames 4096 --steps 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > $O/check.json
