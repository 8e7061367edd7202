set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_redchain.py -q -p no:cacheprovider > gpurun_out/pytest_rc.log 2>&1; tail -30 gpurun_out/pytest_rc.log
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_fusion.py tests/test_gpu_models.py -x -q -p no:cacheprovider > gpurun_out/pytest_g.log 2>&1; tail -5 gpurun_out/pytest_g.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-400
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/graph_launches.csv python tools/profile_step.py 2 graph > gpurun_out/ncu_graph.log 2>&1
tail -2 gpurun_out/ncu_graph.log
