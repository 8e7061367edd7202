timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_ops.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 400 python tools/conv_table.py 2>&1 | tail -1 | cut -c1-100
bash tools/gpu_r2o.sh
