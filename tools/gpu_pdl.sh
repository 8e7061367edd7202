set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_models.py -x -q > gpurun_out/pytest_pdl.log 2>&1; tail -3 gpurun_out/pytest_pdl.log
timeout 300 python tools/launch_gap.py
PB_PDL=0 timeout 300 python tools/launch_gap.py
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-700
PB_PDL=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_nopdl.log 2>&1; tail -1 gpurun_out/bench_nopdl.log | cut -c1-300
