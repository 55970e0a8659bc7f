#!/bin/bash
# fp64 parity window: tile-size sweep (both units see SL_WIN64_T) + profile
out=gpurun_out/r3g; mkdir -p $out
b() { tag=$1; shift; r=$(timeout 300 python bench.py --steps 500 --warmup 10 --no-e2e --no-cpu-baseline --no-fp64 "$@" 2>/dev/null | tail -1); echo "$tag $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"])' 2>&1 | tail -1)" | tee -a $out/sweep.txt; }
b fp64_T12 --precision fp64
bash tools/gpu_prof2.sh r3g fp64 > /dev/null 2>&1
for t in 8 11 14; do
  SL_NVCC_sl_kernels_fp64="-DSL_WIN64_T=$t" SL_NVCC_sl_api="-DSL_WIN64_T=$t" python -c "import sys; sys.path.insert(0,'.'); from paper_1911_10274_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  b fp64_T$t --precision fp64
done
