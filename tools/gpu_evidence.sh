#!/bin/bash
# Round evidence on one B200: gpu tests, default bench line (e2e + CPU
# baseline), reference arm, config D, mixed / fp64 / atomic lines, the ncu
# launch list of the default bench command and one --set full capture of the
# dominant kernel.   usage (via gpurun): bash tools/gpu_evidence.sh TAG
tag=${1:-dev}
out=gpurun_out; mkdir -p $out
python -m pytest tests -m gpu -q 2>&1 | tail -3 > $out/pytest_$tag.txt
cat $out/pytest_$tag.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee $out/smoke_$tag.txt
python bench.py 2>&1 | tail -1 | tee $out/bench_$tag.json
python bench.py --impl reference --steps 3 --warmup 1 2>&1 | tail -1 | tee $out/bench_ref_$tag.json
python bench.py --config D --steps 300 --warmup 10 2>&1 | tail -1 | tee $out/bench_D_$tag.json
python bench.py --config A --steps 2000 --warmup 10 2>&1 | tail -1 | tee $out/bench_A_$tag.json
python bench.py --config A --precision fp64 --steps 2000 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | tee $out/bench_A_fp64_$tag.json
python bench.py --steps 300 --warmup 10 --precision mixed --no-e2e --no-cpu-baseline 2>&1 | tail -1 | tee $out/bench_mixed_$tag.json
python bench.py --steps 100 --warmup 5 --precision fp64 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | tee $out/bench_fp64_$tag.json
python bench.py --steps 100 --warmup 5 --accumulation atomic --no-e2e --no-cpu-baseline 2>&1 | tail -1 | tee $out/bench_atomic_$tag.json
SL_DISABLE_WIN=1 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | tee $out/bench_split_$tag.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file $out/launches_$tag.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
# the step kernels only (3 warm-up + 10 timed steps; the setup launches are
# in launches_TAG)
ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"k_win_tma|k_fused|k_split_step|k_split_tma|k_gather|k_spring|k_mass" -c 100 --csv \
    --log-file $out/launches_timed_$tag.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_win_tma -s 6 -c 1 \
    -o $out/prof_$tag -f python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $out/ncu_full_$tag.log 2>&1
tail -1 $out/ncu_full_$tag.log
for p in fp64 mixed; do
  ncu --set full --clock-control none --import-source on -k regex:k_win_tma -s 6 -c 1 \
      -o $out/prof_${p}_$tag -f python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --precision $p > $out/ncu_full_${p}_$tag.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_fused_small -s 1 -c 1 \
    -o $out/prof_fused_$tag -f python bench.py --config D --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $out/ncu_full_fused_$tag.log 2>&1
python bench.py --n 200 --steps 200 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | tee $out/bench_n200_$tag.json
