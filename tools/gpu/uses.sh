# PB_FUSE_USES default 2: full GPU suite, smoke, bench; 1 and 3 beside it
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "uses=2 $(tail -1 gpurun_out/bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["launches_per_step"], d["e2e"]["value"])')"
for u in 1 3; do PB_FUSE_USES=$u timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_u$u.log 2>&1; echo "uses=$u $(tail -1 gpurun_out/bench_u$u.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["launches_per_step"])')"; done
