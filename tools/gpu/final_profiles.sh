# final profiles at HEAD: five configs, per-kernel time + DRAM of one graph replay
mkdir -p gpurun_out
timeout 600 python tools/bench_configs.py 10 > gpurun_out/bench_configs.jsonl 2>&1; cut -c1-160 gpurun_out/bench_configs.jsonl
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/graph_launches.csv python tools/profile_step.py 2 graph > gpurun_out/ncu_graph.log 2>&1
python tools/bytes_summary.py gpurun_out/graph_launches.csv 100000 > gpurun_out/graph_bytes.txt; head -3 gpurun_out/graph_bytes.txt; gzip -f gpurun_out/graph_launches.csv
