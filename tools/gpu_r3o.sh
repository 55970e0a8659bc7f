#!/bin/bash
out=gpurun_out/r3o; mkdir -p $out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchscale.py tests/test_gpu_window.py tests/test_gpu_fuzz.py tests/test_gpu_goldens_diag.py tests/test_gpu_edge.py tests/test_gpu_control.py -q -x 2>&1 | tail -4 > $out/pytest.txt
cat $out/pytest.txt
b() { tag=$1; shift; r=$(timeout 300 python bench.py --steps 1000 --warmup 20 --no-e2e --no-cpu-baseline --no-fp64 "$@" 2>/dev/null | tail -1); echo "$tag $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"])' 2>&1 | tail -1)" | tee -a $out/sweep.txt; }
b fp64 --precision fp64
b mixed --precision mixed
bash tools/sweep_win4.sh r3o
