# conv routing crossovers re-measured with the round-2 TMA kernel: 1x1 pixel limit and forced TMA wgrad
run() { env $1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cv.log 2>&1;
        echo "$1 $(tail -1 gpurun_out/bench_cv.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["ms_per_step"])')"; }
run "PB_NONE=1"
run "PB_TMA_1X1_MAXPIX=200000"
run "PB_TMA_WGRAD=2"
run "PB_TMA_1X1_MAXPIX=200000 PB_TMA_WGRAD=2"
run "PB_TMA_1X1_MAXPIX=50176"
