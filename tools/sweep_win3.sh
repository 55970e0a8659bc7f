#!/bin/bash
out=gpurun_out/sweep_win3; mkdir -p $out
run() { tag=$1; shift; SL_NVCC_sl_kernels_fp32="$*" python -c "import sys; sys.path.insert(0,'.'); from paper_1911_10274_b200 import _build; _build.build()" > $out/build_$tag.log 2>&1
  for T in 12 16; do SL_WIN_T=$T timeout 300 python bench.py --steps 1000 --warmup 20 --no-e2e --no-cpu-baseline --no-fp64 > $out/b.json 2>&1
  echo "$tag T=$T -> $(python -c "
import json
l=[x for x in open('$out/b.json') if x.startswith('{')]
print(round(json.loads(l[-1])['ms_per_step']*1e3,2) if l else 'fail')") us"; done; }
run base ""
run merged "-DSL_WIN_MERGED"
