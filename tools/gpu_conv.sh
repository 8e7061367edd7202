set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_ops.py -x -q -k "conv" > gpurun_out/pytest_conv.log 2>&1; tail -3 gpurun_out/pytest_conv.log
timeout 300 python tools/conv_table.py > gpurun_out/conv_table.txt 2>&1; tail -27 gpurun_out/conv_table.txt
PB_TMA_1X1=1 timeout 300 python tools/conv_table.py > gpurun_out/conv_table_1x1.txt 2>&1; tail -27 gpurun_out/conv_table_1x1.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
