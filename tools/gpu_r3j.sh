#!/bin/bash
out=gpurun_out/r3j; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_control.py -q -x 2>&1 | tail -3 > $out/pytest.txt
cat $out/pytest.txt
timeout 600 python tools/e2e_steady.py --steps 20 > $out/e2e_steady20.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $out/bench20.json 2>$out/bench20.err
tail -8 $out/e2e_steady20.txt
python -c "import json;d=json.load(open('$out/bench20.json'));print('e2e',d['e2e']['value'],d['e2e']['wall_s'],'dev',d['value'])"
