"""Time fused elementwise chains (GpuBackend(fuse=True)) against the same primitives unfused,
on BatchNorm-shaped operands: GB/s of the algorithmic traffic (leaves read + result written)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2201_12465_b200 import _tensor as T  # noqa: E402
from paper_2201_12465_b200 import registry  # noqa: E402
from paper_2201_12465_b200.gpu.backend import GpuBackend  # noqa: E402

plain = registry.get("gpu")
fused = GpuBackend(name="gpu-fused", fuse=True)
registry.register(fused)
r = np.random.default_rng(0)
shape = (32, 256, 56, 56)
hx = r.standard_normal(shape).astype(np.float32)
hg = r.standard_normal(shape).astype(np.float32)
hc = r.standard_normal((1, 256, 1, 1)).astype(np.float32)
n = hx.size


def programs(be):
    x, g = T.tensor(hx, backend=be.name), T.tensor(hg, backend=be.name)
    c1, c2 = T.tensor(hc, backend=be.name), T.tensor(hc + 1, backend=be.name)
    return {
        "x*c1+c2 (bn affine)": (lambda: (x * c1 + c2).force(), 3),
        "(x-c1)/c2*c1+c2": (lambda: ((x - c1) / c2 * c1 + c2).force(), 5),
        "g*astype(!(x<0)) (relu bwd)": (lambda: (g * x.lt(0.0).logical_not().astype("f32")).force(), 3),
        "x*g+g (2 leaves)": (lambda: (x * g + g).force(), 3),
        "neg(x)": (lambda: x.neg().force(), 2),
    }


for name in programs(plain):
    row = []
    for be in (plain, fused):
        fn, _ = programs(be)[name]
        for _ in range(3):
            fn()
        stop = be.event_timer()
        for _ in range(10):
            fn()
        row.append(stop() / 10)
    leaves = 2 if "g" in name.split("(")[0] else 1
    nbytes = (leaves + 1) * n * 4
    print(f"{name:32s} unfused {row[0]*1e3:8.1f} us  fused {row[1]*1e3:8.1f} us  fused {nbytes / row[1] / 1e6:6.0f} GB/s")
