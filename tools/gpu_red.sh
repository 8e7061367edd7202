set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ops.py -x -q -k "sum or mean or reduce or max or argmax" > gpurun_out/pytest_red.log 2>&1; tail -3 gpurun_out/pytest_red.log
timeout 300 python tools/red_table.py > gpurun_out/red_table.txt 2>&1; cat gpurun_out/red_table.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
