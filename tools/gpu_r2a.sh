#!/bin/bash
# Round-2 first GPU pass: full gpu suite, smoke, bench lines for the window
# tile sizes with compensated fp32 positions.
out=gpurun_out/r2a
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 2>&1 | tail -40 > $out/pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1
for T in 16 12; do
  SL_WIN_INFO=1 SL_WIN_T=$T timeout 300 python bench.py --steps 2000 --warmup 20 --no-e2e --no-cpu-baseline > $out/bench_T$T.json 2> $out/bench_T$T.err
done
timeout 300 python bench.py --steps 20 --warmup 5 > $out/bench_default20.json 2> $out/bench_default20.err
timeout 300 python bench.py --precision mixed --steps 500 --warmup 10 --no-e2e --no-cpu-baseline > $out/bench_mixed.json 2>&1
timeout 300 python bench.py --precision fp64 --steps 500 --warmup 10 --no-e2e --no-cpu-baseline > $out/bench_fp64.json 2>&1
timeout 300 python bench.py --config D --steps 300 --warmup 10 --no-e2e --no-cpu-baseline > $out/bench_D.json 2>&1
tail -3 $out/pytest.txt
