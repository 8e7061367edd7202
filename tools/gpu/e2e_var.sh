# e2e variance: the diagnostic's variants repeated 3x in one process-run each, with SM clocks sampled
for i in 1 2 3; do
  nvidia-smi --query-gpu=clocks.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv,noheader
  timeout 600 python tools/e2e_diag.py 2>&1 | grep -v "^$" | head -8
done
