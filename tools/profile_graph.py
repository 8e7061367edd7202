"""Build the ResNet-50 b32 CapturedStep (traced + planned fusion unless --nofuse) and replay
it N times -- the unit that ncu launch lists of the graph are captured over."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2201_12465_b200 import models, optim, registry, training

be = registry.get("gpu")
be.seed(0)
model = models.resnet50(backend=be.name)
opt = optim.SGD(model.params(), lr=0.01, momentum=0.9)
step = training.CapturedStep(model, opt, warmup=2, fuse="--nofuse" not in sys.argv)
r = np.random.default_rng(0)
x = r.standard_normal((32, 3, 224, 224)).astype(np.float32)
y = r.integers(0, 1000, 32).astype(np.int64)
for _ in range(3):
    step(x, y)
be.synchronize()
n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 1
for _ in range(n):
    step.graph.launch()
be.synchronize()
print("launches/step", step.launches, "fused ops", step.fused_ops)
