"""Golden checkpoint written by the REFERENCE (minml) in the build container.

    python tests/golden/make_checkpoint_golden.py

A small network covering every registered module kind (conv2d, batch_norm, relu,
max_pool2d, view, dropout, linear, log_softmax inside a sequential) trains 2 SGD(momentum)
steps on the reference's eager CPU backend, then minml.training.save_checkpoint writes
checkpoint.mnck (committed).  tests/test_checkpoint.py loads it through this framework and
re-saves it: the bytes must match.  Needs /root/reference; never runs on the GPU box.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from minml import _tensor as MT  # noqa: E402
from minml import nn as MN, optim as MOpt, registry as MR, training as MTr  # noqa: E402
from minml.eager import EagerBackend  # noqa: E402


def net(backend):
    return MN.Sequential(MN.Conv2D(1, 4, 3, backend=backend), MN.BatchNorm(4, backend=backend), MN.ReLU(),
                         MN.MaxPool2D(2), MN.View((4 * 5 * 5,)), MN.Dropout(0.25),
                         MN.Linear(100, 10, backend=backend), MN.LogSoftmax())


be = EagerBackend(name="golden-ckpt", seed=7)
MR.register(be)
model = net(be.name)
opt = MOpt.SGD(model.params(), lr=0.05, momentum=0.9)
r = np.random.default_rng(3)
x = r.standard_normal((6, 1, 12, 12)).astype(np.float32)
y = r.integers(0, 10, 6).astype(np.int64)
for _ in range(2):
    MTr.train_step(model, x, y, opt)
MTr.save_checkpoint(os.path.join(HERE, "checkpoint.mnck"), model, opt, epoch=2, extra={"note": "golden"})
print("wrote", os.path.getsize(os.path.join(HERE, "checkpoint.mnck")), "bytes")
