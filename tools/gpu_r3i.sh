#!/bin/bash
out=gpurun_out/r3i; mkdir -p $out
timeout 600 python tools/e2e_steady.py --steps 20 > $out/e2e_steady20.txt 2>&1
timeout 600 python tools/e2e_steady.py --steps 20 --config D > $out/e2e_steady20_D.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $out/bench20.json 2>$out/bench20.err
timeout 600 python bench.py --config D --steps 20 --warmup 5 --no-cpu-baseline > $out/benchD20.json 2>>$out/bench20.err
cat $out/e2e_steady20.txt | tail -30
