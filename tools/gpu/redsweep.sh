# stage-at-a-time reductions: red_rows rows per block (divisor) and red_cols4s/red_cols4 threshold sweep
for cfg in "1 512" "2 512" "4 512" "1 256" "1 1024"; do
  set -- $cfg
  PB_RED_ROWS_DIV=$1 PB_RED_COLS_THR=$2 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_red_$1_$2.log 2>&1
  echo "rows_div=$1 cols_thr=$2 $(tail -1 gpurun_out/bench_red_$1_$2.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')"
done
