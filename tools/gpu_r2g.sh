out=gpurun_out/r2g; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 -x 2>&1 | tail -30 > $out/pytest.txt
tail -5 $out/pytest.txt
