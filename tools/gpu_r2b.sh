out=gpurun_out/r2b; mkdir -p $out
SL_SKIP_200=0 timeout 900 python -m pytest tests/test_gpu_benchscale.py tests/test_gpu_partition.py -q -s -rf --timeout 800 > $out/pytest.txt 2>&1
tail -5 $out/pytest.txt
