out=gpurun_out/r2n; mkdir -p $out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_win_tma -s 6 -c 1 -o $out/prof_fp64 -f python bench.py --precision fp64 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $out/ncu_fp64.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_win_tma -s 6 -c 1 -o $out/prof_mixed -f python bench.py --precision mixed --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $out/ncu_mixed.log 2>&1
