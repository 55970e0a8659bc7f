out=gpurun_out/r2f; mkdir -p $out
timeout 300 python bench.py --steps 20 --warmup 5 > $out/bench_20.json 2> $out/bench_20.err
timeout 300 python bench.py > $out/bench_default.json 2> $out/bench_default.err
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > $out/ref_20.json 2> $out/ref_20.err
tail -c 2500 $out/bench_20.json; tail -c 600 $out/ref_20.json
