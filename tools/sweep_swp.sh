#!/bin/bash
# fp32 window loop: software-pipelined pair loads vs unrolled pairs
out=gpurun_out/${1:-swp}; mkdir -p $out
b() { tag=$1; shift; r=$(timeout 300 python bench.py --steps 1000 --warmup 20 --no-e2e --no-cpu-baseline --no-fp64 "$@" 2>/dev/null | tail -1); echo "$tag $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"])' 2>&1 | tail -1)" | tee -a $out/sweep.txt; }
for v in "-DWIN_SWP=0 -DWIN_PU=2" "-DWIN_SWP=1" "-DWIN_SWP=0 -DWIN_PU=1"; do
  SL_NVCC_sl_kernels_fp32="$v" python -c "import sys; sys.path.insert(0,'.'); from paper_1911_10274_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  b "$v"
  b "$v" 
done
python -c "import sys; sys.path.insert(0,'.'); from paper_1911_10274_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
