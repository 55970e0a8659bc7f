#!/bin/bash
# split fallback U / warps sweep (SL_DISABLE_WIN=1), fp64 atomic gather
# after batching, and the atomic-path GPU tests
out=gpurun_out/r3u; mkdir -p $out
for u in 4 8 13; do for w in 8 12 16; do
  r=$(SL_DISABLE_WIN=1 SL_SPLIT_U=$u SL_SPLIT_WARPS=$w timeout 300 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu-baseline --no-fp64 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])" 2>&1 | tail -1)
  echo "U=$u W=$w $r" | tee -a $out/sweep_split.txt
done; done
timeout 300 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu-baseline --no-fp64 --precision fp64 --accumulation atomic > $out/b_atomic64.json 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "atomic or auto or fuzz or yield or break" > $out/tests.txt 2>&1
tail -n 2 $out/tests.txt
timeout 600 python tools/e2e_trace.py --steps 20 --config D > $out/e2e_trace_D20.txt 2>&1
