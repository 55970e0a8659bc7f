out=gpurun_out/r2m; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 2>&1 | tail -30 > $out/pytest.txt
tail -4 $out/pytest.txt
timeout 300 python bench.py --steps 20 --warmup 5 > $out/bench_20.json 2> $out/bench_20.err
timeout 300 python bench.py > $out/bench_default.json 2> $out/bench_default.err
timeout 300 python tools/e2e_breakdown.py --steps 20 > $out/e2e_bd.txt 2>&1
