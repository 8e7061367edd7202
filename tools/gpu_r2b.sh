set -x
mkdir -p gpurun_out
rm -f gpurun_out/fullsize_parity.jsonl
timeout 900 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_graph.py tests/test_gpu_minml_dropin.py -x -q > gpurun_out/pytest_new.log 2>&1; tail -15 gpurun_out/pytest_new.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q > gpurun_out/pytest_full.log 2>&1; tail -15 gpurun_out/pytest_full.log
cat gpurun_out/fullsize_parity.jsonl | cut -c1-250
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-3000
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-300
