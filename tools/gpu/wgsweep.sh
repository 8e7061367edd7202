# wgrad routing re-measured: 1x1 GEMM path for every shape (PB_WG_MM=2), TMA wgrad up to 56x56 (PB_TMA_WG_P2)
run() { env $1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_wg.log 2>&1;
        echo "$1 $(tail -1 gpurun_out/bench_wg.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["ms_by_kind"])')"; }
run "PB_NONE=1"
run "PB_WG_MM=2"
run "PB_TMA_WG_P2=100352"
run "PB_WG_MM=2 PB_TMA_WG_P2=100352"
