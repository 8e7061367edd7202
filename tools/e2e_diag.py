"""Where does the pipelined e2e step (CapturedStep.run) lose time against graph-only replay?
ResNet-50 b32, page-locked batch; CUDA events + wall clock per variant (diagnostic only)."""
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
x = be.pinned((32, 3, 224, 224), np.float32)
x[...] = r.standard_normal((32, 3, 224, 224)).astype(np.float32)
y = be.pinned((32,), np.int64)
y[...] = r.integers(0, 1000, 32)
step = training.CapturedStep(model, opt, warmup=2)
for _ in range(4):
    step(x, y)
list(step.run([(x, y)] * 2))
be.synchronize()
K = 20


def timed(name, fn):
    be.synchronize()
    t0 = time.perf_counter()
    stop = be.event_timer()
    fn()
    ms = stop() / K
    print(f"{name:44s} events {ms:7.3f} ms  wall {(time.perf_counter() - t0) * 1e3 / K:7.3f} ms", flush=True)


timed("graph only", lambda: [step.graph.launch() for _ in range(K)])
timed("step(x, y) (sync per step)", lambda: [step(x, y) for _ in range(K)])
timed("run() pipelined", lambda: list(step.run([(x, y)] * K)))


def h2d_only():
    for _ in range(K):
        be.stage_in(step.x, x, stream=2)
        be.stream_sync(2)


timed("stage_in x on copy stream + sync", h2d_only)


def graph_plus_copystream():
    for _ in range(K):
        be.stage_in(step._stage[0][0], x, stream=2)
        step.graph.launch()
    be.stream_sync(2)


timed("graph + concurrent copy-stream H2D", graph_plus_copystream)
