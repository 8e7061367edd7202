"""Device cost of a tiny dependent kernel inside a CUDA graph: record K chained elementwise
adds on a small vector, replay, time per kernel (diagnostic for the step's ~1.8k tiny
launches)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2201_12465_b200 import _tensor as T  # noqa: E402
from paper_2201_12465_b200 import registry  # noqa: E402

be = registry.get("gpu")
for n in (256, 65536, 1 << 20):
    x = T.tensor(np.ones(n, np.float32), backend=be.name)
    y = T.tensor(np.ones(n, np.float32), backend=be.name)
    K = 1000
    be.capture_begin()
    keep = []
    v = x
    for _ in range(K):
        v = v + y
        keep.append(v)
    g = be.capture_end()
    for _ in range(3):
        g.launch()
    stop = be.event_timer()
    for _ in range(5):
        g.launch()
    ms = stop() / 5
    print(f"n={n:8d}: {ms * 1e3 / K:6.2f} us per chained kernel in a graph", flush=True)
