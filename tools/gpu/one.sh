# one-step reduction sources: parity, bench A/B (PB_RC_INTERP=1), launch list
mkdir -p gpurun_out; rm -f gpurun_out/*.ncu-rep
timeout 900 python -m pytest tests/test_gpu_redchain.py tests/test_gpu_graph.py tests/test_gpu_fullsize.py tests/test_gpu_models.py -x -q > gpurun_out/pytest_one.log 2>&1; tail -2 gpurun_out/pytest_one.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_one.log 2>&1; tail -1 gpurun_out/bench_one.log | cut -c1-250
PB_RC_INTERP=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_one_interp.log 2>&1; tail -1 gpurun_out/bench_one_interp.log | cut -c1-250
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_one.csv python tools/profile_step.py 2 graph > gpurun_out/ncu_launch.log 2>&1
python tools/graph_breakdown.py gpurun_out/launches_one.csv 100000 > gpurun_out/launches_one.txt; grep -i red gpurun_out/launches_one.txt
