out=gpurun_out/r2h; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 2>&1 | tail -40 > $out/pytest.txt
tail -12 $out/pytest.txt
