# e2e after pre-allocating every posted-read slot: pipelined tests, bench x4 (a fresh process each)
timeout 600 python -m pytest tests/test_gpu_graph.py tests/test_gpu_runtime.py -x -q > gpurun_out/pytest_pipe.log 2>&1; tail -1 gpurun_out/pytest_pipe.log
for i in 1 2 3 4; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_p.log 2>&1; tail -1 gpurun_out/bench_p.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("bench", d["ms_per_step"], d["e2e"]["ms_per_step"], d["e2e"]["value"])'; done
