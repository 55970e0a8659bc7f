#!/bin/bash
# fp32 window kernel (entry words): pair-unroll x tile-size sweep, config B
out=gpurun_out/${1:-sw4}; mkdir -p $out
b() { tag=$1; shift; r=$(timeout 300 python bench.py --steps 1000 --warmup 20 --no-e2e --no-cpu-baseline --no-fp64 "$@" 2>/dev/null | tail -1); echo "$tag $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"])' 2>&1 | tail -1)" | tee -a $out/sweep.txt; }
for pu in 1 2 3; do
  SL_NVCC_sl_kernels_fp32="-DWIN_PU=$pu" python -c "import sys; sys.path.insert(0,'.'); from paper_1911_10274_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  b PU${pu}_T16
  SL_WIN_T=12 b PU${pu}_T12
  SL_WIN_T=10 b PU${pu}_T10
done
python -c "import sys; sys.path.insert(0,'.'); from paper_1911_10274_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
