set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_models.py tests/test_gpu_graph.py tests/test_gpu_fusion.py -x -q > gpurun_out/pytest_pad.log 2>&1; tail -3 gpurun_out/pytest_pad.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-250
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/graph_launches.csv python tools/profile_step.py 2 graph > gpurun_out/ncu_graph.log 2>&1
python tools/bytes_summary.py gpurun_out/graph_launches.csv 2900 > gpurun_out/graph_bytes.txt; grep "pad_fast\|launches," gpurun_out/graph_bytes.txt
