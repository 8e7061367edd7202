set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_ops.py tests/test_gpu_models.py tests/test_gpu_graph.py -x -q > gpurun_out/pytest_ws.log 2>&1; tail -3 gpurun_out/pytest_ws.log
timeout 300 python tools/conv_table.py > gpurun_out/conv_table.txt 2>&1; tail -1 gpurun_out/conv_table.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-250
