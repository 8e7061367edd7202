timeout 300 python -m pytest tests/test_gpu_models.py -x -q 2>&1 | grep -E "assert|Error|passed|failed" | head -8
timeout 600 python tools/conv_table.py 2>&1 | tail -30
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_iter.log 2>&1; tail -1 gpurun_out/bench_iter.log | cut -c1-300
