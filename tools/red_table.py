"""Time the reduction shapes of a ResNet-50 b32 step (BatchNorm statistics and the
_unbroadcast sums of its backward) with CUDA events: achieved GB/s per shape."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2201_12465_b200 import _tensor as T  # noqa: E402
from paper_2201_12465_b200 import registry  # noqa: E402

be = registry.get("gpu")
r = np.random.default_rng(0)
CASES = []
for c, h in ((64, 112), (64, 56), (256, 56), (128, 28), (512, 28), (256, 14), (1024, 14), (512, 7), (2048, 7)):
    CASES += [((32, c, h, h), 3), ((32, c, h), 2), ((32, c), 0), ((32, c, h, h), 0), ((1, c, h, h), 2),
              ((1, c, 1, h), 3)]
print(f"{'shape':>22} ax | {'us':>8} {'GB/s':>7}")
tot = 0.0
for shape, ax in CASES:
    x = T.tensor(r.standard_normal(shape).astype(np.float32), backend=be.name)
    for _ in range(3):
        x.sum(axis=ax, keepdims=True)
    reps = 20
    stop = be.event_timer()
    for _ in range(reps):
        x.sum(axis=ax, keepdims=True)
    ms = stop() / reps
    nbytes = int(np.prod(shape)) * 4
    tot += ms
    print(f"{str(shape):>22} {ax:2d} | {ms * 1e3:8.2f} {nbytes / ms / 1e6:7.0f}")
print(f"sum {tot:.3f} ms")
