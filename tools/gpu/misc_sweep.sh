# existing policy hooks re-measured at HEAD: all reduction chains fused (PB_RC_ALL), chains recomputed by 2 consumers (PB_FUSE_USES=2)
run() { env $1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_ms.log 2>&1;
        echo "$1 $(tail -1 gpurun_out/bench_ms.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["launches_per_step"])')"; }
run "PB_NONE=1"
run "PB_RC_ALL=1"
run "PB_FUSE_USES=2"
