timeout 1200 python -m pytest tests/test_gpu_fusion.py tests/test_gpu_graph.py tests/test_gpu_window.py tests/test_gpu_redchain.py -q -x -p no:cacheprovider 2>&1 | tail -3
bash tools/gpu_r2o.sh
