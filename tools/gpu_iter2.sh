set -x
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_ops.py -x -q 2>&1 | tail -4
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_iter.log 2>&1; tail -1 gpurun_out/bench_iter.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches3.csv python tools/profile_step.py 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches3.csv 4500 | head -40
