#!/bin/bash
# Theta-tile raster groups (AMLT_THETA_GROUP_ROWS) against DRAM traffic and
# time: ncu dram bytes of one launch on 4096 rows of config 4, and the pinned
# bench at full size. Scratch experiment (traffic).
out=gpurun_out/raster; mkdir -p $out
T=discount_f64_48x128_theta_t6x4_w8x1
for g in 480 960 1776 3552; do
  AMLT_THETA_GROUP_ROWS=$g timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --kernel-name-base demangled -k regex:BodyTheta -c 1 --csv --page raw --log-file $out/g$g.csv \
    python tools/profile_one.py discount f64 4096 8192 32768 $T > $out/g$g.log 2>&1
  echo "g=$g ncu rc=$?"
  [ -n "$NO_BENCH" ] || AMLT_THETA_GROUP_ROWS=$g python bench.py --tile $T --steps 3 --warmup 1 --no-e2e --no-cpu --no-verify > $out/bench_g$g.json 2>/dev/null
  python -c "import json; d=json.load(open('$out/bench_g$g.json')); print('g=$g', d['ms_per_step'])"
done
