#!/bin/bash
# multi-step window launches: targeted tests, then bench fp32 / mixed / fp64
# against SL_NO_MULTISTEP=1
out=gpurun_out/r3p; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_benchscale.py tests/test_gpu_parity.py -q -x 2>&1 | tail -15 > $out/pytest1.txt
cat $out/pytest1.txt
b() { tag=$1; shift; r=$(timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-fp64 "$@" 2>/dev/null | tail -1); echo "$tag $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["call_ms_per_step"], d["roofline"]["frac"])' 2>&1 | tail -1)" | tee -a $out/sweep.txt; }
for p in fp32 mixed fp64; do
  b ${p}_multi_1000 --precision $p --steps 1000 --warmup 20
  SL_NO_MULTISTEP=1 b ${p}_single_1000 --precision $p --steps 1000 --warmup 20
  b ${p}_multi_20 --precision $p --steps 20 --warmup 5
  SL_NO_MULTISTEP=1 b ${p}_single_20 --precision $p --steps 20 --warmup 5
done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -6 > $out/pytest.txt
cat $out/pytest.txt
