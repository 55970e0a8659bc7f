#!/bin/bash
out=gpurun_out/r3s; mkdir -p $out
for w in 2 4 8; do
  for r in 1 2; do
  SL_E2E_WARM=$w timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-fp64 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('warm $w', d['e2e']['value'], d['e2e']['wall_s'])" | tee -a $out/e2e.txt
  done
done
