# chain taps: parity (fusion/graph/fullsize/redchain/window), bench A/B against PB_FUSE_TAPS=0, launch list
mkdir -p gpurun_out; rm -f gpurun_out/*.ncu-rep
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_fusion.py tests/test_gpu_fullsize.py tests/test_gpu_redchain.py tests/test_gpu_window.py tests/test_gpu_models.py -x -q > gpurun_out/pytest_taps.log 2>&1; tail -5 gpurun_out/pytest_taps.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_taps.log 2>&1; tail -1 gpurun_out/bench_taps.log | cut -c1-250
PB_FUSE_TAPS=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_notaps.log 2>&1; tail -1 gpurun_out/bench_notaps.log | cut -c1-250
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_taps.csv python tools/profile_step.py 2 graph > gpurun_out/ncu_launch.log 2>&1
python tools/bytes_summary.py gpurun_out/launches_taps.csv 100000 | head -12
