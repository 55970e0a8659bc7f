#!/bin/bash
# Sweep the window kernel's window stages (SL_WIN_WS) and slice slots.
out=gpurun_out; mkdir -p $out
for cfg in ${CFGS:-"2 64" "3 64" "4 64" "3 18" "3 14"}; do
  set -- $cfg
  r=$(SL_WIN_WS=$1 SL_WIN_SLOTS=$2 timeout 120 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline "${@:3}" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['frac'],3), d['roofline']['kernel'])")
  echo "WS=$1 SLOTS<=$2 $r" | tee -a $out/sweep_win_$TAG.txt
done
