out=gpurun_out/r2c; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 -s 2>&1 > $out/pytest.txt
grep -E "passed|failed|config" $out/pytest.txt | tail -8
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1
timeout 300 python bench.py --steps 2000 --warmup 20 --no-e2e --no-cpu-baseline > $out/bench_B.json 2>&1
timeout 300 python bench.py --config D --steps 300 --warmup 10 --no-e2e --no-cpu-baseline > $out/bench_D.json 2>&1
