"""Run W warm-up + 1 ResNet-50 b32 training step (device-resident batch) — the unit that
ncu launch lists in profiles/ are captured over."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2201_12465_b200 as pb  # noqa: F401
from paper_2201_12465_b200 import _tensor as T
from paper_2201_12465_b200 import models, nn, optim, registry
from paper_2201_12465_b200.autograd import Variable

be = registry.get("gpu")
model = models.resnet50(backend=be.name)
opt = optim.SGD(model.params(), lr=0.01, momentum=0.9)
rng = np.random.default_rng(0)
x = Variable(T.tensor(rng.standard_normal((32, 3, 224, 224)).astype(np.float32), backend=be.name))
y = T.tensor(rng.integers(0, 1000, 32).astype(np.int64), backend=be.name)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
if len(sys.argv) > 2 and sys.argv[2] == "graph":
    # captured step (fused plan): warm-up + record, then ONE replay -- the last
    # launches_per_step kernels of an ncu launch list over this command are that replay
    from paper_2201_12465_b200 import training
    xh = rng.standard_normal((32, 3, 224, 224)).astype(np.float32)
    yh = rng.integers(0, 1000, 32).astype(np.int64)
    step = training.CapturedStep(model, opt, warmup=2)
    for _ in range(3):
        step(xh, yh)
    be.synchronize()
    # only the replay is profiled (ncu --profile-from-start off)
    import ctypes
    cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
    if cudart is not None:
        cudart.cudaProfilerStart()
    step.graph.launch()
    be.synchronize()
    if cudart is not None:
        cudart.cudaProfilerStop()
    print("graph launches per step", step.launches)
    sys.exit(0)
for _ in range(steps):
    opt.zero_grad()
    loss = nn.cross_entropy(model(x), y)
    loss.backward()
    opt.step()
be.synchronize()
print("loss", loss.scalar(), "launches", be.launch_count())
