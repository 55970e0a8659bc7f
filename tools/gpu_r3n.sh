#!/bin/bash
out=gpurun_out/r3n; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_control.py -q -x 2>&1 | tail -15 > $out/pytest_ctl.txt
cat $out/pytest_ctl.txt
timeout 600 python tools/predicate_bench.py 2>&1 | tail -6 | tee $out/predicate.txt
