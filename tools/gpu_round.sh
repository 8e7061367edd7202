set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-400
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-300
timeout 600 python tools/conv_table.py > gpurun_out/conv_table.txt 2>&1; tail -3 gpurun_out/conv_table.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py 2 > gpurun_out/ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 4500 > gpurun_out/launches.txt; head -40 gpurun_out/launches.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tma -c 3 -o gpurun_out/conv_full -f python tools/conv_once.py 32 64 56 56 64 3 1 1 > gpurun_out/ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/conv_full.ncu-rep > gpurun_out/conv_full.txt 2>&1; head -40 gpurun_out/conv_full.txt
