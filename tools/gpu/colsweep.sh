# cols-mode reduction chain: (row, column-unit) pairs per block sweep, device ms per step
for pairs in 256 128 64 512; do
  PB_RC_COLS_PAIRS=$pairs timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cols_$pairs.log 2>&1
  echo "pairs=$pairs $(tail -1 gpurun_out/bench_cols_$pairs.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')"
done
