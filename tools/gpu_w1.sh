timeout 600 python -m pytest tests/test_gpu_window.py -q -x -p no:cacheprovider 2>&1 | tail -25
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_fusion.py tests/test_gpu_redchain.py tests/test_gpu_models.py -q -x -p no:cacheprovider 2>&1 | tail -3
