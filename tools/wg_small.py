"""One wgrad through the TMA path vs SIMT: python tools/wg_small.py N C H W F K pad"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2201_12465_b200 import _tensor as T, registry
be = registry.get("gpu")
n, c, h, w, f, k, p = [int(v) for v in sys.argv[1:8]]
r = np.random.default_rng(0)
xs, ws = (n, c, h, w), (f, c, k, k)
ho, wo = h + 2 * p - k + 1, w + 2 * p - k + 1
x = T.tensor(r.standard_normal(xs).astype(np.float32), backend=be.name)
g = T.tensor(r.standard_normal((n, f, ho, wo)).astype(np.float32), backend=be.name)
a = T.conv2d_grad_weight(x, g, ws, 1, p).to_host_buffer()
be._lib.pb_set_gemm_path(0)
b = T.conv2d_grad_weight(x, g, ws, 1, p).to_host_buffer().astype(np.float64)
d = np.abs(a - b) / np.maximum(np.abs(b), 1)
print("case", sys.argv[1:8], "max rel", d.max(), "bad", int((d > 1e-5).sum()), "of", d.size)
