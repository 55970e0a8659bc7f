#!/bin/bash
# One GPU round trip: tests, bench lines, launch list, one full ncu capture.
# usage (via gpurun): bash tools/gpu_check.sh [tag] [ncu:0/1] [kernel-regex]
tag=${1:-dev}
do_ncu=${2:-1}
kre=${3:-k_split_tma}
out=gpurun_out
mkdir -p $out
python -m pytest tests -m gpu -q -rA 2>&1 | grep -E "passed|failed|FAILED|Error|error|assert" | tail -60 > $out/pytest_$tag.txt
cat $out/pytest_$tag.txt
python bench.py --steps 300 --warmup 10 2>&1 | tail -1 | tee $out/bench_$tag.json
SL_DISABLE_SPLIT=1 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | tee $out/bench_exact_$tag.json
python bench.py --steps 300 --warmup 10 --precision mixed --no-e2e --no-cpu-baseline 2>&1 | tail -1 | tee $out/bench_mixed_$tag.json
python bench.py --steps 100 --warmup 5 --precision fp64 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | tee $out/bench_fp64_$tag.json
python bench.py --steps 100 --warmup 5 --accumulation atomic --no-e2e --no-cpu-baseline 2>&1 | tail -1 | tee $out/bench_atomic_$tag.json
if [ "$do_ncu" = "1" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file $out/launches_$tag.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:$kre -s 6 -c 1 \
    -o $out/prof_$tag -f python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $out/ncu_full_$tag.log 2>&1
tail -2 $out/ncu_full_$tag.log
fi
