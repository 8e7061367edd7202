# warp-rows reduction chains: parity tests, bench A/B against the plane-staged kernel (PB_RC_STAGED=1), launch list
mkdir -p gpurun_out; rm -f gpurun_out/*.ncu-rep
timeout 900 python -m pytest tests/test_gpu_redchain.py tests/test_gpu_fusion.py tests/test_gpu_graph.py tests/test_gpu_window.py -x -q > gpurun_out/pytest_rows.log 2>&1; tail -2 gpurun_out/pytest_rows.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_rows.log 2>&1; tail -1 gpurun_out/bench_rows.log | cut -c1-250
PB_RC_STAGED=1 timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_staged.log 2>&1; tail -1 gpurun_out/bench_staged.log | cut -c1-250
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rows.csv python tools/profile_step.py 2 graph > gpurun_out/ncu_launch.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_fullsize.log 2>&1; tail -2 gpurun_out/pytest_fullsize.log
