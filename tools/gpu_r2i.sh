out=gpurun_out/r2i; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_halo.py tests/test_gpu_partition.py -q -rf --timeout 600 -x 2>&1 | tail -30 > $out/pytest.txt
tail -5 $out/pytest.txt
timeout 600 python bench.py --config E --steps 50 --warmup 5 > $out/bench_E1.json 2> $out/bench_E1.err
tail -c 400 $out/bench_E1.json
BENCH_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --config E --edge 100 --gpus 2 --steps 10 --warmup 3 > $out/bench_E2.json 2> $out/bench_E2.err
tail -c 600 $out/bench_E2.json; tail -5 $out/bench_E2.err
