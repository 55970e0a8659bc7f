#!/bin/bash
out=gpurun_out/r3l; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > $out/pytest.txt
cat $out/pytest.txt
timeout 600 python tools/e2e_settle.py --steps 20 2>&1 | tail -30 > $out/settle.txt
grep "^rep" $out/settle.txt
for c in B D; do
timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_$c.json 2>$out/bench_$c.err
python -c "import json;d=json.load(open('$out/bench_$c.json'));print('$c e2e',d['e2e']['value'],d['e2e']['wall_s'],'dev',d['value'])"
done
