#!/bin/bash
out=gpurun_out/r3r; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_benchscale.py tests/test_gpu_window.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3 > $out/pytest.txt
cat $out/pytest.txt
b() { tag=$1; shift; r=$(timeout 300 python bench.py --steps 1000 --warmup 20 --no-e2e --no-cpu-baseline --no-fp64 "$@" 2>/dev/null | tail -1); echo "$tag $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"])' 2>&1 | tail -1)" | tee -a $out/sweep.txt; }
b fp32; b fp32; b fp32_20 --steps 20 --warmup 5
