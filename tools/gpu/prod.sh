# product-source reduction chains: parity, bench A/B against the interpreter (PB_RC_INTERP=1), launch list
mkdir -p gpurun_out; rm -f gpurun_out/*.ncu-rep
timeout 900 python -m pytest tests/test_gpu_redchain.py tests/test_gpu_fusion.py tests/test_gpu_graph.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_prod.log 2>&1; tail -2 gpurun_out/pytest_prod.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_prod.log 2>&1; tail -1 gpurun_out/bench_prod.log | cut -c1-250
PB_RC_INTERP=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_interp.log 2>&1; tail -1 gpurun_out/bench_interp.log | cut -c1-250
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_prod.csv python tools/profile_step.py 2 graph > gpurun_out/ncu_launch.log 2>&1
python tools/graph_breakdown.py gpurun_out/launches_prod.csv 2379 | grep -i "red\|launches"
