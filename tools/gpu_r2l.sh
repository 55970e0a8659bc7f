out=gpurun_out/r2l; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 2>&1 | tail -30 > $out/pytest.txt
tail -4 $out/pytest.txt
timeout 900 python tools/hub_sweep.py fp32 > $out/hub_fp32.jsonl 2> $out/hub_fp32.err
timeout 900 python tools/hub_sweep.py fp64 > $out/hub_fp64.jsonl 2> $out/hub_fp64.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_split_atomic -s 3 -c 1 -o $out/prof_atomic -f python bench.py --accumulation atomic --steps 6 --warmup 3 --no-e2e --no-cpu-baseline --no-fp64 > $out/ncu_atomic.log 2>&1
SL_ATOMIC_KERNEL=spring timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spring_atomic -s 3 -c 1 -o $out/prof_spring -f python bench.py --accumulation atomic --steps 6 --warmup 3 --no-e2e --no-cpu-baseline --no-fp64 > $out/ncu_spring.log 2>&1
