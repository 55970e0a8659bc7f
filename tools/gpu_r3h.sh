#!/bin/bash
# fp64 parity window: (tile, interleave) sweep with the host unit in sync
out=gpurun_out/r3h; mkdir -p $out
b() { tag=$1; shift; r=$(timeout 300 python bench.py --steps 500 --warmup 10 --no-e2e --no-cpu-baseline --no-fp64 "$@" 2>/dev/null | tail -1); echo "$tag $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"])' 2>&1 | tail -1)" | tee -a $out/sweep.txt; }
for v in "12 2" "11 3" "11 4" "7 4" "7 6" "9 4"; do
  set -- $v
  SL_NVCC_sl_kernels_fp64="-DSL_WIN64_T=$1 -DWIN_XU=$2" SL_NVCC_sl_api="-DSL_WIN64_T=$1" python -c "import sys; sys.path.insert(0,'.'); from paper_1911_10274_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  b fp64_T$1_XU$2 --precision fp64
done
