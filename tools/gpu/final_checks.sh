# JIT chain grid sweep (waves of resident blocks), then compute-sanitizer memcheck over the round-2 kernels
mkdir -p gpurun_out
for w in 1 2 0; do
  PB_JIT_WAVES=$w timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_waves_$w.log 2>&1
  echo "jit_waves=$w $(tail -1 gpurun_out/bench_waves_$w.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')"
done
timeout 1200 compute-sanitizer --tool memcheck --leak-check none --error-exitcode 9 python -m pytest -x -q tests/test_gpu_redchain.py "tests/test_gpu_graph.py::test_chain_taps_bit_identical_and_fewer_launches" tests/test_gpu_window.py > gpurun_out/sanitizer_round2.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/sanitizer_round2.log
