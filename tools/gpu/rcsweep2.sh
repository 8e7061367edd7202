# rows-mode plane budget around the chosen 48 KB, at HEAD defaults
for kb in 48 32 64 40; do
  PB_RC_SMEM_KB=$kb timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_kb.log 2>&1
  echo "smem_kb=$kb $(tail -1 gpurun_out/bench_kb.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["e2e"]["ms_per_step"])')"
done
