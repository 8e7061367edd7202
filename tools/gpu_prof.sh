set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/graph_launches.csv python tools/profile_step.py 2 graph > gpurun_out/ncu_graph.log 2>&1
tail -2 gpurun_out/ncu_graph.log
python tools/bytes_summary.py gpurun_out/graph_launches.csv 2905 > gpurun_out/graph_bytes.txt; cat gpurun_out/graph_bytes.txt
timeout 300 python tools/red_table.py > gpurun_out/red_table.txt 2>&1; cat gpurun_out/red_table.txt
