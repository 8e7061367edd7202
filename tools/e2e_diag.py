"""Where does the e2e step lose time against graph-only replay?  Times ResNet-50 b32
CapturedStep variants with wall clock + CUDA events (diagnostic only)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2201_12465_b200 import models, optim, registry, training  # noqa: E402

be = registry.get("gpu")
be.seed(0)
model = models.resnet50(backend=be.name)
opt = optim.SGD(model.params(), lr=0.01, momentum=0.9)
r = np.random.default_rng(0)
x = r.standard_normal((32, 3, 224, 224)).astype(np.float32)
y = r.integers(0, 1000, 32).astype(np.int64)
step = training.CapturedStep(model, opt, warmup=2)
for _ in range(4):
    step(x, y)
be.synchronize()
K = 10


def timed(name, fn):
    be.synchronize()
    t0 = time.perf_counter()
    stop = be.event_timer()
    for _ in range(K):
        fn()
    ms = stop() / K
    print(f"{name:40s} events {ms:7.3f} ms  wall {(time.perf_counter() - t0) * 1e3 / K:7.3f} ms", flush=True)


timed("graph only", lambda: step.graph.launch())
timed("copy_in x,y (compute stream)", lambda: (be.copy_in(step.x, x), be.copy_in(step.y, y)))
timed("graph + copy_in", lambda: (be.copy_in(step.x, x), be.copy_in(step.y, y), step.graph.launch()))
timed("graph + loss.scalar", lambda: (step.graph.launch(), step.loss.scalar()))
timed("step(x, y)", lambda: step(x, y))
sx = be  # noqa
t0 = time.perf_counter()
for _ in range(K):
    np.ascontiguousarray(x).copy()
print(f"host copy of x: {(time.perf_counter() - t0) * 1e3 / K:.3f} ms")
be.synchronize()
t0 = time.perf_counter()
stop = be.event_timer()
n = len(list(step.run([(x, y)] * K)))
print(f"run() x{n}: events {stop() / K:.3f} ms wall {(time.perf_counter() - t0) * 1e3 / K:.3f} ms")
