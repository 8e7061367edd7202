# rows-mode reduction chain: planes per block (shared-memory budget / block target) sweep, device ms per step
for cfg in "96 4" "48 4" "24 4" "48 8" "24 16" "12 16"; do
  set -- $cfg
  PB_RC_SMEM_KB=$1 PB_RC_TARGET=$2 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_rc_$1_$2.log 2>&1
  echo "smem_kb=$1 target=$2 $(tail -1 gpurun_out/bench_rc_$1_$2.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')"
done
