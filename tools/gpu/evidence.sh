# Round evidence on one B200: GPU tests, smoke, both bench arms, five configs, conv table,
# per-kernel time+DRAM of one graph replay, and an ncu --set full capture of the step's top conv.
set -x
mkdir -p gpurun_out; rm -f gpurun_out/*.ncu-rep
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-300
timeout 600 python tools/bench_configs.py 10 > gpurun_out/bench_configs.jsonl 2>&1; cut -c1-200 gpurun_out/bench_configs.jsonl
timeout 600 python tools/conv_table.py > gpurun_out/conv_table.txt 2>&1; tail -3 gpurun_out/conv_table.txt
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/graph_launches.csv python tools/profile_step.py 2 graph > gpurun_out/ncu_graph.log 2>&1
python tools/bytes_summary.py gpurun_out/graph_launches.csv 100000 > gpurun_out/graph_bytes.txt; head -30 gpurun_out/graph_bytes.txt; gzip -f gpurun_out/graph_launches.csv
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:tma_conv_kernel -c 1 -o gpurun_out/conv_step_full -f python tools/profile_step.py 2 graph > gpurun_out/ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/conv_step_full.ncu-rep > gpurun_out/conv_step_full.txt 2>&1; head -20 gpurun_out/conv_step_full.txt
