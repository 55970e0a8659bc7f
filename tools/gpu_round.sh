set -x
bash tools/gpu_check.sh r1h 1 k_split_tma
python bench.py --config D --steps 300 --warmup 10 2>&1 | tail -1 | tee gpurun_out/bench_D_r1h.json
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee gpurun_out/smoke_r1h.txt
