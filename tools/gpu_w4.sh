timeout 600 python -m pytest tests/test_gpu_window.py tests/test_gpu_graph.py -q -x -p no:cacheprovider 2>&1 | tail -2
bash tools/gpu_r2o.sh
