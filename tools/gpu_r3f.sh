#!/bin/bash
# velocity staging + fp64 interleave sweep (config B)
out=gpurun_out/r3f; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchscale.py tests/test_gpu_window.py tests/test_gpu_fused.py tests/test_gpu_edge.py -q -x 2>&1 | tail -4 > $out/pytest.txt
cat $out/pytest.txt
b() { tag=$1; shift; r=$(timeout 300 python bench.py --steps 1000 --warmup 10 --no-e2e --no-cpu-baseline --no-fp64 "$@" 2>/dev/null | tail -1); echo "$tag $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"])' 2>&1 | tail -1)" | tee -a $out/sweep.txt; }
b fp32 --precision fp32
SL_WIN_VSTAGE=1 b fp32_vst --precision fp32
b mixed_vst --precision mixed
SL_WIN_VSTAGE=0 b mixed_reg --precision mixed
b fp64_xu2 --precision fp64
for xu in 3 4; do
  SL_NVCC_sl_kernels_fp64="-DWIN_XU=$xu" python -c "import sys; sys.path.insert(0,'.'); from paper_1911_10274_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  b fp64_xu$xu --precision fp64
done
