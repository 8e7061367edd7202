set -x
mkdir -p gpurun_out
rm -f gpurun_out/fullsize_parity.jsonl
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_all.log 2>&1; tail -30 gpurun_out/pytest_all.log
cut -c1-300 gpurun_out/fullsize_parity.jsonl
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-3000
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-600
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/graph_launches.csv python tools/profile_step.py 2 graph > gpurun_out/ncu_graph.log 2>&1
python tools/bytes_summary.py gpurun_out/graph_launches.csv 2900 > gpurun_out/graph_bytes.txt; head -45 gpurun_out/graph_bytes.txt
