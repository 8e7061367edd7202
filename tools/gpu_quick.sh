set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_graph.py tests/test_abi_cpu.py -x -q > gpurun_out/pytest_graph.log 2>&1; tail -15 gpurun_out/pytest_graph.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -3 gpurun_out/bench.log | cut -c1-1500
