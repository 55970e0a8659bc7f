#!/bin/bash
# Fast GPU iteration: gpu tests, the default bench line, one ncu capture.
# usage (via gpurun): bash tools/gpu_quick.sh tag [kernel-regex] [bench args]
tag=${1:-dev}
kre=${2:-k_split_tma}
shift 2
out=gpurun_out
mkdir -p $out
python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > $out/pytest_$tag.txt
cat $out/pytest_$tag.txt
python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline "$@" 2>&1 | tail -1 | tee $out/bench_$tag.json
ncu --set full --clock-control none --import-source on -k regex:$kre -s 6 -c 1 \
    -o $out/prof_$tag -f python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" > $out/ncu_full_$tag.log 2>&1
tail -2 $out/ncu_full_$tag.log
