set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python tools/conv_table.py > gpurun_out/conv_table.txt 2>&1; tail -27 gpurun_out/conv_table.txt
PB_TMA_WGRAD=2 PB_TMA_1X1=1 timeout 300 python tools/conv_table.py > gpurun_out/conv_table_all.txt 2>&1; tail -27 gpurun_out/conv_table_all.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-400
