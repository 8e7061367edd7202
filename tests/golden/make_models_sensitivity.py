"""The reference's own conditioning for the reduced trajectories of models.json: each config
rerun by minml from an init perturbed by 1e-7 (relative, about one f32 ulp), recording how far
its losses and per-parameter sums move.  tests/test_gpu_models.py allows twice that where it
exceeds the 1e-3 bar (the batch-4 BatchNorm ResNet is chaotic: a 1e-7 nudge moves its
cancelling signed weight sums by ~1e-2).

    PB_NO_AUTOREGISTER=1 python tests/golden/make_models_sensitivity.py   ->  models_sensitivity.json
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
os.environ.setdefault("PB_NO_AUTOREGISTER", "1")

from minml import _tensor as MT, autograd as MA, nn as MN, ops as MO  # noqa: E402
from minml import optim as MOpt, registry as MR, training as MTr  # noqa: E402
from minml.eager import EagerBackend  # noqa: E402

from paper_2201_12465_b200 import models as PM  # noqa: E402

sys.path.insert(0, HERE)
import inputs as GI  # noqa: E402

NS = PM.namespace(MN, MO, MT, MA)
BUILD = {
    "mlp": lambda be: PM.mlp(784, 256, 10, backend=be, ns=NS),
    "lenet": lambda be: PM.mnist_cnn(backend=be, ns=NS),
    "alexnet_tiny": lambda be: PM.alexnet(classes=10, image=67, channels=(8, 16, 24, 16, 16), hidden=64, backend=be,
                                          ns=NS),
    "resnet_tiny": lambda be: PM.resnet50(classes=10, layers=(1, 1, 1, 1), width=8, backend=be, ns=NS),
    "bert_tiny": lambda be: PM.bert_base(vocab=50, seq=8, d=16, heads=2, ffn=32, layers=2, classes=2, backend=be,
                                         ns=NS),
}


def run(name, meta, perturb):
    be_name = f"sens-{name}-{perturb}"
    MR.register(EagerBackend(name=be_name, seed=meta["seed"]))
    try:
        model = BUILD[name](be_name)
        if perturb:
            r = np.random.default_rng(1)
            for p in model.params():
                a = p.numpy()
                p.data = MT.tensor((a * (1 + perturb * r.standard_normal(a.shape))).astype(a.dtype), backend=be_name)
        opt = MOpt.SGD(model.params(), **meta["sgd"])
        if name == "bert_tiny":
            bs = [GI.batch(name, k, None, 2, meta["batch"], tokens=(meta["seq"], meta["vocab"])) for k in range(2)]
        else:
            bs = [GI.batch(name, k, tuple(meta["input"]), meta["classes"], meta["batch"]) for k in range(2)]
        losses = [float(MTr.train_step(model, *bs[k % 2], opt)[0]) for k in range(meta["steps"])]
        sums = [[float(np.sum(p.numpy(), dtype=np.float64)), float(np.sum(np.abs(p.numpy()), dtype=np.float64))]
                for p in model.params()]
    finally:
        MR.unregister(be_name)
    return losses, sums


def main():
    with open(os.path.join(HERE, "models.json")) as f:
        meta = json.load(f)
    out = {}
    rel = lambda u, v: abs(u - v) / max(abs(u), abs(v), 1.0)  # noqa: E731
    for name in BUILD:
        l0, s0 = run(name, meta[name], 0.0)
        assert l0 == meta[name]["losses"], name  # the unperturbed rerun reproduces the golden
        l1, s1 = run(name, meta[name], 1e-7)
        out[name] = {"loss": max(rel(u, v) for u, v in zip(l0, l1)),
                     "sums": max(max(rel(a[0], b[0]), rel(a[1], b[1])) for a, b in zip(s0, s1))}
        print(name, out[name], flush=True)
    with open(os.path.join(HERE, "models_sensitivity.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
