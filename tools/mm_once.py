"""One rank-2 matmul x @ W^T through the backend -- a short target for ncu --set full
captures of the TMA GEMM (`-k regex:tma_conv`).    python tools/mm_once.py [M K N]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2201_12465_b200 import _tensor as T  # noqa: E402
from paper_2201_12465_b200 import registry  # noqa: E402

M, K, N = [int(v) for v in sys.argv[1:]] or [2048, 3072, 768]
be = registry.get("gpu")
r = np.random.default_rng(0)
x = T.tensor(r.standard_normal((M, K)).astype(np.float32), backend=be.name)
w = T.tensor((r.standard_normal((N, K)) * 0.02).astype(np.float32), backend=be.name)
y = T.matmul(x, w.transpose())
be.synchronize()
print("ok", y.shape)
