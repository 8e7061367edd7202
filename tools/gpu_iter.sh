# quick iteration: contraction parity tests, per-shape conv table, bench (no CPU baseline)
set -x
timeout 900 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -5
timeout 600 python tools/conv_table.py 2>&1 | tail -30
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_iter.log 2>&1; tail -1 gpurun_out/bench_iter.log | cut -c1-400
