# PB_FUSE_USES=2 re-measured with the 3-deep pipelined run: bench x3 (device, e2e pipelined, e2e one call)
for i in 1 2 3; do PB_FUSE_USES=2 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_u2.log 2>&1; tail -1 gpurun_out/bench_u2.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["e2e"]; print("uses=2", d["ms_per_step"], e["ms_per_step"], e["unpipelined"]["ms_per_step"], d["launches_per_step"])'; done
for i in 1 2; do PB_FUSE_USES=2 timeout 600 python tools/e2e_diag.py 2>&1 | grep "pipelined\|graph only"; done
