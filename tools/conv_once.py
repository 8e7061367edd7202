"""Run one ResNet-50 conv (fprop, dgrad, wgrad) through the backend -- a short target for
``ncu --set full -k regex:tc_gemm`` captures.

    python tools/conv_once.py [N C H W F KH stride pad]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2201_12465_b200 import _tensor as T  # noqa: E402
from paper_2201_12465_b200 import registry  # noqa: E402

a = [int(v) for v in sys.argv[1:]] or [32, 64, 56, 56, 64, 3, 1, 1]
n, c, h, w, f, k, s, p = a
be = registry.get("gpu")
r = np.random.default_rng(0)
x = T.tensor(r.standard_normal((n, c, h, w)).astype(np.float32), backend=be.name)
wt = T.tensor((r.standard_normal((f, c, k, k)) * 0.05).astype(np.float32), backend=be.name)
y = T.conv2d(x, wt, None, s, p)
g = T.tensor(r.standard_normal(tuple(y.shape)).astype(np.float32), backend=be.name)
T.conv2d_grad_input(g, wt, (n, c, h, w), s, p)
T.conv2d_grad_weight(x, g, (f, c, k, k), s, p)
be.synchronize()
print("ok")
