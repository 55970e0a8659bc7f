#!/bin/bash
out=gpurun_out/r3q; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_benchscale.py -q -x 2>&1 | tail -3 > $out/pytest1.txt
cat $out/pytest1.txt
b() { tag=$1; shift; r=$(timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-fp64 "$@" 2>/dev/null | tail -1); echo "$tag $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["call_ms_per_step"], d["roofline"]["frac"])' 2>&1 | tail -1)" | tee -a $out/sweep.txt; }
for p in fp32 fp64; do
  b ${p}_multi_1000 --precision $p --steps 1000 --warmup 20
  SL_NO_MULTISTEP=1 b ${p}_single_1000 --precision $p --steps 1000 --warmup 20
done
