# reduction tap (BatchNorm's c = x - mu stored by the variance reduction): parity, bench A/B, launch list
mkdir -p gpurun_out; rm -f gpurun_out/*.ncu-rep
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_redchain.py tests/test_gpu_fullsize.py tests/test_gpu_fusion.py tests/test_gpu_models.py -x -q > gpurun_out/pytest_rtap.log 2>&1; tail -3 gpurun_out/pytest_rtap.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_rtap.log 2>&1; echo "rtap $(tail -1 gpurun_out/bench_rtap.log | cut -c1-230)"
PB_FUSE_TAPS=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_rtap_off.log 2>&1; echo "taps off $(tail -1 gpurun_out/bench_rtap_off.log | cut -c1-230)"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_rtap.csv python tools/profile_step.py 2 graph > gpurun_out/ncu_launch.log 2>&1
python tools/bytes_summary.py gpurun_out/launches_rtap.csv 100000 > gpurun_out/graph_bytes_rtap.txt; head -14 gpurun_out/graph_bytes_rtap.txt
