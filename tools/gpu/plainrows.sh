PB_RC_PLAIN_ROWS=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_plainrows.log 2>&1; echo "plain_rows $(tail -1 gpurun_out/bench_plainrows.log | cut -c1-300)"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_default.log 2>&1; echo "default $(tail -1 gpurun_out/bench_default.log | cut -c1-300)"
