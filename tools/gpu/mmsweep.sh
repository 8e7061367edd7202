# matmul routing re-measured: TMA-fed matmul down to M = 64 (AlexNet's classifier at b128, BERT) vs the default M >= 256
for m in 256 128 64; do
  PB_TMA_MM_MIN_M=$m timeout 600 python tools/bench_configs.py 10 mlp alexnet bert > gpurun_out/cfg_mm_$m.jsonl 2>&1
  echo "min_m=$m"; python -c "
import json
for l in open('gpurun_out/cfg_mm_$m.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print('  ', d['config'], round(d['device']['ms_per_step'],3))"
done
