#!/bin/bash
# fp32 window kernel (compensated positions): tile slices x ring stages, and
# the stream-only experiment (SL_WIN_DBG=1: copies, no force computation)
out=gpurun_out/sweep_win2; mkdir -p $out
run() { SL_WIN_INFO=1 env "$@" timeout 300 python bench.py --steps 1000 --warmup 20 --no-e2e --no-cpu-baseline --no-fp64 > $out/b.json 2> $out/b.err;
  echo "$* -> $(python -c "
import json
l=[x for x in open('$out/b.json') if x.startswith('{')]
print(round(json.loads(l[-1])['ms_per_step']*1e3,2) if l else 'fail')") us  $(grep -o '[0-9]* stages' $out/b.err | tail -1)"; }
run SL_WIN_T=12
run SL_WIN_T=12 SL_WIN_STAGES=2
run SL_WIN_T=16
run SL_WIN_T=8
run SL_WIN_T=8 SL_WIN_STAGES=2
run SL_WIN_T=20
run SL_WIN_T=12 SL_WIN_DBG=1
run SL_WIN_T=16 SL_WIN_DBG=1
run SL_WIN_T=8 SL_WIN_DBG=1
