#!/bin/bash
# fp64 parity window kernel: tile slices x interleaved entries (WIN_XU).
# Each variant rebuilds libsoftlat_cuda.so (both units see the macros).
out=gpurun_out/sweep_fp64; mkdir -p $out
for v in "12 2" "11 2" "11 3" "11 4" "8 3" "8 4"; do
  set -- $v
  flags="-DSL_WIN64_T=$1 -DWIN_XU=$2"
  SL_NVCC_sl_kernels_fp64="$flags" SL_NVCC_sl_api="$flags" python -c "import sys; sys.path.insert(0,'.'); from paper_1911_10274_b200 import _build; _build.build()" > $out/build_$1_$2.log 2>&1
  timeout 300 python bench.py --precision fp64 --steps 300 --warmup 10 --no-e2e --no-cpu-baseline > $out/bench_$1_$2.json 2>&1
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "fp64_gather" 2>&1 | tail -1 > $out/parity_$1_$2.txt
  echo "T=$1 XU=$2 $(tail -c 300 $out/bench_$1_$2.json | grep -o '"ms_per_step": [0-9.]*') $(cat $out/parity_$1_$2.txt)"
done
