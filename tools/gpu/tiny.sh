# tiny-chain batching + ragged windowed chains: targeted tests, then the bench A/B (PB_TINY_BATCH=0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fusion.py tests/test_gpu_graph.py tests/test_gpu_window.py -x -q > gpurun_out/pytest_tiny.log 2>&1; tail -3 gpurun_out/pytest_tiny.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_tiny.log 2>&1; tail -1 gpurun_out/bench_tiny.log | cut -c1-250
PB_TINY_BATCH=0 timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_notiny.log 2>&1; tail -1 gpurun_out/bench_notiny.log | cut -c1-250
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tiny.csv python tools/profile_step.py 2 graph > gpurun_out/ncu_launch.log 2>&1
