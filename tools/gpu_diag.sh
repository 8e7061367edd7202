timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_iter.log 2>&1; tail -1 gpurun_out/bench_iter.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['launches_per_step'], d.get('fused_ops'), d.get('graph_error'))"
