#!/bin/bash
# Sweep the window kernel's tile slices T and ring depth (tile stages).
# usage: CFGS="16:4 12:4" TAG=x bash tools/sweep_win.sh [bench args]
out=gpurun_out; mkdir -p $out
for cfg in ${CFGS:-16:4 16:3 16:2 12:4}; do
  t=${cfg%%:*}; s=${cfg##*:}
  r=$(SL_WIN_T=$t SL_WIN_STAGES=$s timeout 120 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['frac'],3), d['roofline']['kernel'])")
  echo "T=$t S=$s $r" | tee -a $out/sweep_win_$TAG.txt
done
