mkdir -p gpurun_out
rm -f gpurun_out/fullsize_parity.jsonl
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_all.log 2>&1; tail -25 gpurun_out/pytest_all.log
cut -c1-330 gpurun_out/fullsize_parity.jsonl
timeout 300 python tools/fprop_bias_diag.py > gpurun_out/fprop_bias.txt 2>&1; cat gpurun_out/fprop_bias.txt
timeout 300 python tools/conv_table.py > gpurun_out/conv_table.txt 2>&1; tail -22 gpurun_out/conv_table.txt
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-1500
