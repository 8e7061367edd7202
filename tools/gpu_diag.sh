timeout 600 python -m pytest tests/test_gpu_ops.py -x -q 2>&1 | tail -2
timeout 300 python tools/red_table.py 2>&1 | grep -E " 3 \||sum"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_iter.log 2>&1; tail -1 gpurun_out/bench_iter.log | cut -c1-250
