#!/bin/bash
# ncu --set full of one fused step kernel of a bench workload
# usage: bash tools/gpu_prof.sh TAG KERNEL_REGEX [bench args...]
tag=$1; kre=$2; shift 2
out=gpurun_out; mkdir -p $out
ncu --set full --clock-control none --import-source on -k regex:$kre -s ${SKIP:-6} -c 1 \
    -o $out/prof_$tag -f python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" > $out/ncu_full_$tag.log 2>&1
tail -2 $out/ncu_full_$tag.log
