mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_ops.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 400 python tools/conv_table.py > gpurun_out/conv_table.txt 2>&1; tail -26 gpurun_out/conv_table.txt
