#!/bin/bash
# atomic step's mass pass (k_mass): what its 57 us go to (diagnostic
# variants; MASS_NOPLANES changes the physics and is timing-only)
out=gpurun_out/${1:-mass}; mkdir -p $out
b() { tag=$1; shift; r=$(timeout 300 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline --no-fp64 --accumulation atomic "$@" 2>/dev/null | tail -1); echo "$tag $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])' 2>&1 | tail -1)" | tee -a $out/sweep.txt; }
l() { tag=$1; timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_mass -c 5 --csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-fp64 --accumulation atomic 2>/dev/null | grep k_mass | tail -2 | sed "s/^/$tag /" >> $out/sweep.txt; }
for v in "" "-DMASS_NOSTOP" "-DMASS_NOPLANES" "-DMASS_NOSTOP -DMASS_NOPLANES"; do
  SL_NVCC_sl_kernels_fp32="$v" python -c "import sys; sys.path.insert(0,'.'); from paper_1911_10274_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  b "[$v]"
  l "[$v]"
done
SL_PDL=0 b "[SL_PDL=0]"
python -c "import sys; sys.path.insert(0,'.'); from paper_1911_10274_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
