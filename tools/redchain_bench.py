"""Time pb_reduce_chain on ResNet-50 b32 BatchNorm shapes (fwd mean chain, bwd sum chain of a
plain tensor and of a 2-leaf product) against the one-kernel-per-stage path; GB/s of the
algorithmic bytes (every leaf read once)."""
import os
import struct
import sys

os.environ["PB_RC_ALL"] = "1"

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2201_12465_b200 import _tensor as T, registry
from paper_2201_12465_b200.gpu import _lib

be = registry.get("gpu")
lib = _lib.load()
SHAPES = [(32, 64, 112, 112), (32, 64, 56, 56), (32, 256, 56, 56), (32, 128, 28, 28), (32, 256, 28, 28), (32, 512, 28, 28),
          (32, 256, 14, 14), (32, 1024, 14, 14), (32, 512, 7, 7), (32, 2048, 7, 7)]


def timeit(fn, reps=20):
    """Device time per call: `reps` calls recorded into a CUDA graph, replayed (no host gaps)."""
    fn()
    be.synchronize()
    be.capture_begin()
    for _ in range(reps):
        fn()
    graph = be.capture_end()
    graph.launch()
    be.synchronize()
    t = be.event_timer()
    graph.launch()
    ms = t()
    return ms / reps * 1e3


def chain(leaves, steps, shape, stages, out):
    lv = b"".join(l.adapter.packed() for l in leaves)
    sp = b"".join(_lib.STEP.pack(*s) for s in steps)
    stg = b"".join(_lib.RSTAGE.pack(*s) for s in stages)
    rc = lib.pb_reduce_chain(len(leaves), lv, 0, 0.0, len(steps), sp, 4, struct.pack("<4q", *shape), len(stages),
                             stg, out.adapter.packed())
    _lib.check(rc, "chain")


for shape in SHAPES:
    N, C, H, W = shape
    x = T.tensor(np.random.default_rng(0).standard_normal(shape).astype(np.float32), backend="gpu")
    y = T.tensor(np.random.default_rng(1).standard_normal(shape).astype(np.float32), backend="gpu")
    out = T.tensor(np.zeros((C,), np.float32), backend="gpu")
    nb = x.shape.size * 4
    fwd = [(3, 3, 0, float(W)), (2, 3, 0, float(H)), (0, 3, 0, float(N))]
    bwd = [(0, -1, 0, 0.0), (2, -1, 0, 0.0), (3, -1, 0, 0.0)]
    t_f = timeit(lambda: chain([x], [], shape, fwd, out))
    t_b = timeit(lambda: chain([x], [], shape, bwd, out))
    t_p = timeit(lambda: chain([x, y], [(2, 1, 0, 1, 0, 0, 0.0)], shape, bwd, out))
    sd = T.tensor(np.random.default_rng(2).random((1, C, 1, 1)).astype(np.float32) + 0.5, backend="gpu")
    # neg((x / sd) * y / sd): BatchNorm backward's grad-of-std chain (3 leaves, 2 divisions)
    bn3 = [(3, 1, 0, 2, 0, 0, 0.0), (2, 1, 0, 1, 0, 0, 0.0), (3, 1, 0, 2, 0, 0, 0.0), (64, 0, 0, 0, 0, 0, 0.0)]
    t_b3 = timeit(lambda: chain([x, y, sd], bn3, shape, bwd, out))
    t_sq = timeit(lambda: chain([x], [(2, 3, 0, 0, 0, 0, 0.0)], shape, fwd, out))
    t_old_f = timeit(lambda: x.mean(3).mean(2).mean(0))
    t_old_b = timeit(lambda: x.sum(0, keepdims=True).sum(2, keepdims=True).sum(3, keepdims=True))
    print(f"{str(shape):22s} {nb / 1e6:7.1f} MB | fwd {t_f:7.1f} us {nb / t_f / 1e3:6.0f} GB/s | bwd {t_b:7.1f} us "
          f"{nb / t_b / 1e3:6.0f} GB/s | prod {t_p:7.1f} us {2 * nb / t_p / 1e3:6.0f} GB/s | sq {t_sq:6.1f} | bn3 {t_b3:6.1f} {2 * nb / t_b3 / 1e3:5.0f} GB/s | old fwd {t_old_f:7.1f} "
          f"bwd {t_old_b:7.1f} us", flush=True)
