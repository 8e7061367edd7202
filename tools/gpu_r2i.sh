mkdir -p gpurun_out
timeout 300 python tools/redchain_bench.py 2>&1 | tee gpurun_out/redchain_bench.txt

timeout 600 python -m pytest tests/test_gpu_redchain.py tests/test_gpu_graph.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/graph_launches.csv python tools/profile_step.py 2 graph > gpurun_out/ncu_graph.log 2>&1
python tools/bytes_summary.py gpurun_out/graph_launches.csv 100000 > gpurun_out/graph_bytes.txt; head -30 gpurun_out/graph_bytes.txt; rm -f gpurun_out/graph_launches.csv
