#!/bin/bash
# ncu --set full + source hot list of the window kernel for several precisions
# usage: bash tools/gpu_prof2.sh TAG prec1 [prec2 ...]
tag=$1; shift
for p in "$@"; do
  out=gpurun_out/$tag/$p; mkdir -p $out
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KRE:-k_win_tma} -s 6 -c 1 \
      -o $out/prof -f python bench.py --precision $p --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-fp64 > $out/ncu.log 2>&1
  ncu -i $out/prof.ncu-rep --page source --csv --print-source sass > $out/src.csv 2>/dev/null
  python tools/ncu_summary.py $out/prof.ncu-rep $out/ncu_summary.txt > /dev/null 2>&1
  python tools/ncu_hot.py $out/src.csv 40 > $out/hot.txt 2>&1
  gzip -f $out/src.csv
  head -16 $out/ncu_summary.txt
done
