# quick perf check: config B (fp32), D, and the fp32 parity tests
out=gpurun_out/${1:-q}; mkdir -p $out
timeout 300 python bench.py --steps 2000 --warmup 20 --no-e2e --no-cpu-baseline --no-fp64 > $out/bench_B.json 2>&1
timeout 300 python bench.py --config D --steps 300 --warmup 10 --no-e2e --no-cpu-baseline > $out/bench_D.json 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_window.py tests/test_gpu_fused.py tests/test_gpu_benchscale.py -q -x -k "not 200" 2>&1 | tail -2 > $out/pytest.txt
for f in bench_B bench_D; do python -c "
import json
l=[x for x in open('$out/$f.json') if x.startswith('{')]
d=json.loads(l[-1]); print('$f', round(d['ms_per_step']*1e3,2), '%.3g'%d['value'], round(d['roofline']['frac'],3))"; done
cat $out/pytest.txt
