#!/bin/bash
# ncu --set full of the config-D split kernel + its SASS source page
tag=${1:-d}
out=gpurun_out; mkdir -p $out
ncu --set full --clock-control none --import-source on -k regex:k_split_tma -s 6 -c 1 \
    -o $out/prof_$tag -f python bench.py --config D --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $out/ncu_full_$tag.log 2>&1
tail -2 $out/ncu_full_$tag.log
