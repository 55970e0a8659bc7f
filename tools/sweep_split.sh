#!/bin/bash
# Sweep the split kernel's gather batch U and warps per CTA (fp32, 100^3).
out=gpurun_out; mkdir -p $out
for u in ${US:-4 8 13}; do for w in ${WS:-8 12 16}; do
  r=$(SL_SPLIT_U=$u SL_SPLIT_WARPS=$w python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])")
  echo "U=$u W=$w $r" | tee -a $out/sweep_$TAG.txt
done; done
