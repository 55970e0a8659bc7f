#!/bin/bash
out=gpurun_out/r3m; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_inplace_edits.py -q -x 2>&1 | tail -25 > $out/pytest_inc.txt
cat $out/pytest_inc.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > $out/pytest.txt
cat $out/pytest.txt
