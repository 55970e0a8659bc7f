#!/bin/bash
out=gpurun_out/r3t; mkdir -p $out
for r in 1 2 3; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-fp64 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());e=d['e2e'];print('B', e['value'], e['wall_s'], e['segment_walls_s'])" | tee -a $out/e2e.txt
done
timeout 600 python bench.py --config D --steps 20 --warmup 5 --no-cpu-baseline --no-fp64 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());e=d['e2e'];print('D', e['value'], e['wall_s'], e['segment_walls_s'])" | tee -a $out/e2e.txt
