set -x
timeout 900 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -15
timeout 600 python tools/conv_table.py 2>&1 | tail -30
