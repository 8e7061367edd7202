set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_ops.py -x -q -k "conv or grad_input" > gpurun_out/pytest_dg.log 2>&1; tail -15 gpurun_out/pytest_dg.log
timeout 300 python tools/conv_table.py > gpurun_out/conv_table.txt 2>&1; tail -27 gpurun_out/conv_table.txt
