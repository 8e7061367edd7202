set -x
mkdir -p gpurun_out
timeout 200 python tools/mm_table.py > gpurun_out/mm_table.txt 2>&1; echo "mm_table rc=$?"; tail -3 gpurun_out/mm_table.txt
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_ops.py tests/test_gpu_models.py tests/test_gpu_graph.py -x -q > gpurun_out/pytest_mm.log 2>&1; tail -2 gpurun_out/pytest_mm.log
timeout 600 python tools/bench_configs.py 10 > gpurun_out/bench_configs.jsonl 2>&1; echo "cfg rc=$?"; cut -c1-250 gpurun_out/bench_configs.jsonl
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-250
