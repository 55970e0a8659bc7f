#!/bin/bash
out=gpurun_out/${1:-sw64pu}; mkdir -p $out
b() { tag=$1; shift; r=$(timeout 300 python bench.py --precision fp64 --steps 500 --warmup 10 --no-e2e --no-cpu-baseline --no-fp64 "$@" 2>/dev/null | tail -1); echo "$tag $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"])' 2>&1 | tail -1)" | tee -a $out/sweep.txt; }
for u in 1 2 3; do
  SL_NVCC_sl_kernels_fp64="-DWIN64_PU=$u" python -c "import sys; sys.path.insert(0,'.'); from paper_1911_10274_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  b PU$u; b PU$u
done
python -c "import sys; sys.path.insert(0,'.'); from paper_1911_10274_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
