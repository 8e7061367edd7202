import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
import numpy as np
from frontend_util import BUILDERS
from paper_2201_12465_b200 import optim, training, registry
be = registry.get("gpu")
be.seed(3)
model = BUILDERS["lenet"](be.name)
opt = optim.SGD(model.params(), lr=0.05, momentum=0.9)
r = np.random.default_rng(0)
x = r.standard_normal((4, 1, 28, 28)).astype(np.float32); y = r.integers(0, 10, 4).astype(np.int64)
if "plan" in sys.argv:
    training.train_step(model, x, y, opt)
    be.fusion_trace_begin(); training.train_step(model, x, y, opt); be.fusion_trace_end()
    be.fusion_plan_begin()
    try:
        print(training.train_step(model, x, y, opt)[0])
    finally:
        be.fusion_plan_end()
else:
    step = training.CapturedStep(model, opt, warmup=2, fuse=True)
    for _ in range(4):
        print(step(x, y)[0])
