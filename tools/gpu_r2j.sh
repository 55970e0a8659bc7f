out=gpurun_out/r2j; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_halo.py tests/test_gpu_partition.py -q -rf --timeout 600 2>&1 | tail -30 > $out/pytest.txt
tail -5 $out/pytest.txt
