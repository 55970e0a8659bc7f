timeout 1200 python bench.py --n 200 --steps 500 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_n200_r1k.json
cat gpurun_out/bench_n200_r1k.json | cut -c1-300
