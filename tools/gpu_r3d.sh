#!/bin/bash
out=gpurun_out/r3d; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchscale.py tests/test_gpu_window.py tests/test_gpu_goldens_diag.py tests/test_gpu_edits.py tests/test_gpu_fuzz.py tests/test_gpu_fuzz_edits.py -q -x 2>&1 | tail -6 > $out/pytest.txt
cat $out/pytest.txt
for p in fp32 mixed fp64; do
  timeout 300 python bench.py --precision $p --steps 1000 --warmup 10 --no-e2e --no-cpu-baseline --no-fp64 2>/dev/null | tail -1 > $out/bench_$p.json
  python -c "import json;d=json.load(open('$out/bench_$p.json'));print('$p',d['ms_per_step'],d['value'],d['roofline']['frac'])"
done
bash tools/sweep_fp64b.sh r3d
