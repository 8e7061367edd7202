mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['launches_per_step'], d['e2e']['ms_per_step'], d['roofline']['ms_per_step'], d['roofline']['achieved'])"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/graph_launches.csv python tools/profile_step.py 2 graph > gpurun_out/ncu_graph.log 2>&1
python tools/bytes_summary.py gpurun_out/graph_launches.csv 100000 > gpurun_out/graph_bytes.txt; head -24 gpurun_out/graph_bytes.txt; gzip -f gpurun_out/graph_launches.csv
