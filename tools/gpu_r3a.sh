#!/bin/bash
# Session restart check: GPU tests + the default and 20-step bench lines.
out=gpurun_out/r3a; mkdir -p $out
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > $out/pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1; echo "smoke rc=$?" >> $out/smoke.txt
timeout 900 python bench.py > $out/bench_default.json 2> $out/bench_default.err
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench_n20.json 2> $out/bench_n20.err
tail -3 $out/pytest.txt
