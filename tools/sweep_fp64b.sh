#!/bin/bash
# fp64 parity window kernel: branch-free sqrt / divide; sweep the entry
# interleave (WIN_XU) and the tile size (SL_WIN64_T), bench fp64 config B.
out=gpurun_out/${1:-sw64}; mkdir -p $out
for v in "2 12" "3 12" "4 12" "2 11" "4 11" "3 10"; do
  set -- $v
  export SL_NVCC_sl_kernels_fp64="-DWIN_XU=$1 -DSL_WIN64_T=$2"
  python -c "import sys; sys.path.insert(0,'.'); from paper_1911_10274_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  r=$(timeout 300 python bench.py --precision fp64 --steps 300 --warmup 10 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1)
  echo "XU=$1 T=$2 $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"])' 2>&1)" | tee -a $out/sweep.txt
done
unset SL_NVCC_sl_kernels_fp64
python -c "import sys; sys.path.insert(0,'.'); from paper_1911_10274_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
