# e2e variance with the cyclic GC paused inside CapturedStep.run: diagnostic x3, pipelined-run tests, bench
for i in 1 2 3; do timeout 600 python tools/e2e_diag.py 2>&1 | grep "pipelined\|graph only"; done
timeout 600 python -m pytest tests/test_gpu_graph.py -x -q -k "pipelined or pinned" > gpurun_out/pytest_pipe.log 2>&1; tail -1 gpurun_out/pytest_pipe.log
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_gc.log 2>&1; tail -1 gpurun_out/bench_gc.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("bench", d["ms_per_step"], d["e2e"]["ms_per_step"], d["e2e"]["value"])'; done
