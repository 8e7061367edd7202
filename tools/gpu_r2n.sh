mkdir -p gpurun_out
rm -f gpurun_out/fullsize_parity.jsonl
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_all.log 2>&1; tail -3 gpurun_out/pytest_all.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-400
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/graph_launches.csv python tools/profile_step.py 2 graph > gpurun_out/ncu_graph.log 2>&1
python tools/bytes_summary.py gpurun_out/graph_launches.csv 100000 > gpurun_out/graph_bytes.txt; head -30 gpurun_out/graph_bytes.txt; gzip -f gpurun_out/graph_launches.csv
