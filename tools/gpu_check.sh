#!/bin/bash
# One GPU round trip: tests, bench lines, launch list, one full ncu capture.
# usage (via gpurun): bash tools/gpu_check.sh [tag]
tag=${1:-dev}
out=gpurun_out
mkdir -p $out
python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > $out/pytest_$tag.txt
cat $out/pytest_$tag.txt
python bench.py --steps 300 --warmup 10 2>&1 | tail -1 | tee $out/bench_$tag.json
python bench.py --steps 300 --warmup 10 --precision mixed --no-e2e --no-cpu-baseline 2>&1 | tail -1 | tee $out/bench_mixed_$tag.json
python bench.py --steps 100 --warmup 5 --accumulation atomic --no-e2e --no-cpu-baseline 2>&1 | tail -1 | tee $out/bench_atomic_$tag.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file $out/launches_$tag.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gather_step -s 6 -c 1 \
    -o $out/prof_gather_$tag -f python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $out/ncu_full_$tag.log 2>&1
tail -3 $out/ncu_full_$tag.log
