out=gpurun_out/r2e; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 -s 2>&1 > $out/pytest.txt
grep -E "passed|failed|config" $out/pytest.txt | tail -8
SL_WIN_INFO=1 timeout 300 python bench.py --steps 2000 --warmup 20 --no-e2e --no-cpu-baseline > $out/bench_B.json 2>&1
SL_WIN_T=16 timeout 300 python bench.py --steps 2000 --warmup 20 --no-e2e --no-cpu-baseline > $out/bench_B16.json 2>&1
timeout 300 python bench.py --config D --steps 300 --warmup 10 --no-e2e --no-cpu-baseline > $out/bench_D.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_win_tma -s 6 -c 1 -o $out/prof_win -f python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $out/ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 1 -o $out/prof_fused -f python bench.py --config D --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $out/ncu_d.log 2>&1
