#!/bin/bash
# fp32 window kernel: 1 vs 2 CTAs per SM (smaller tiles, 2 stages each)
out=gpurun_out/${1:-ctas}; mkdir -p $out
b() { tag=$1; shift; r=$(timeout 300 python bench.py --steps 1000 --warmup 20 --no-e2e --no-cpu-baseline --no-fp64 "$@" 2>/dev/null | tail -1); echo "$tag $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"])' 2>&1 | tail -1)" | tee -a $out/sweep.txt; }
b T16_1cta
SL_WIN_T=8 SL_WIN_STAGES=2 SL_WIN_CTAS=2 b T8_2cta_2st
SL_WIN_T=8 SL_WIN_STAGES=3 SL_WIN_CTAS=1 b T8_1cta_3st
SL_WIN_T=8 SL_WIN_STAGES=2 SL_WIN_CTAS=1 b T8_1cta_2st
SL_WIN_T=4 SL_WIN_STAGES=2 SL_WIN_CTAS=3 b T4_3cta
SL_WIN_T=4 SL_WIN_STAGES=3 SL_WIN_CTAS=2 b T4_2cta_3st
b mixed_T12 --precision mixed
SL_WIN_T=8 SL_WIN_STAGES=2 SL_WIN_CTAS=2 b mixed_T8_2cta --precision mixed
