mkdir -p gpurun_out
rm -f gpurun_out/fullsize_parity.jsonl
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_all.log 2>&1; tail -8 gpurun_out/pytest_all.log
cut -c1-200 gpurun_out/fullsize_parity.jsonl
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_smoke.log 2>&1; tail -4 gpurun_out/sanitizer_smoke.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_redchain.py tests/test_gpu_graph.py -q -x -p no:cacheprovider -k "not dropout" > gpurun_out/sanitizer_tests.log 2>&1; tail -4 gpurun_out/sanitizer_tests.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_redchain.py -q -x -p no:cacheprovider > gpurun_out/racecheck_redchain.log 2>&1; tail -4 gpurun_out/racecheck_redchain.log
