timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_ops.py tests/test_gpu_models.py tests/test_gpu_fullsize.py -q -p no:cacheprovider 2>&1 | tail -4
timeout 400 python tools/conv_table.py 2>&1 | tail -1 | cut -c1-100
