set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-200
timeout 300 python tools/conv_table.py > gpurun_out/conv_table.txt 2>&1; tail -1 gpurun_out/conv_table.txt
timeout 600 python tools/bench_configs.py 10 > gpurun_out/bench_configs.jsonl 2>&1; cut -c1-200 gpurun_out/bench_configs.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py 2 graph > gpurun_out/ncu_launch.log 2>&1
python tools/graph_breakdown.py gpurun_out/launches.csv 2900 > gpurun_out/launches.txt 2>&1; head -5 gpurun_out/launches.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tma_conv -c 2 -o gpurun_out/conv_full -f python tools/conv_once.py 32 64 56 56 64 3 1 1 > gpurun_out/ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/conv_full.ncu-rep > gpurun_out/conv_full.txt 2>&1; head -18 gpurun_out/conv_full.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tma_conv -c 1 -o gpurun_out/mm_full -f python tools/mm_once.py 2048 3072 768 > gpurun_out/ncu_mm.log 2>&1
python tools/ncu_summary.py gpurun_out/mm_full.ncu-rep > gpurun_out/mm_full.txt 2>&1; head -18 gpurun_out/mm_full.txt
