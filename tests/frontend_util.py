"""Run the five config families' reduced trajectories through the product front end
on any registered backend (the oracle on CPU, the GPU backend on the box)."""

import numpy as np

import inputs as GI
from paper_2201_12465_b200 import models as PM
from paper_2201_12465_b200 import optim, training

BUILDERS = {
    "mlp": lambda be: PM.mlp(784, 256, 10, backend=be),
    "lenet": lambda be: PM.mnist_cnn(backend=be),
    "alexnet_tiny": lambda be: PM.alexnet(classes=10, image=67, channels=(8, 16, 24, 16, 16), hidden=64, backend=be),
    "resnet_tiny": lambda be: PM.resnet50(classes=10, layers=(1, 1, 1, 1), width=8, backend=be),
    "bert_tiny": lambda be: PM.bert_base(vocab=50, seq=8, d=16, heads=2, ffn=32, layers=2, classes=2, backend=be),
}


def batches(name, meta):
    if name == "bert_tiny":
        return [GI.batch(name, k, None, 2, meta["batch"], tokens=(meta["seq"], meta["vocab"])) for k in range(2)]
    return [GI.batch(name, k, tuple(meta["input"]), meta["classes"], meta["batch"]) for k in range(2)]


def run_trajectory(name, meta, backend):
    backend.seed(meta["seed"])
    model = BUILDERS[name](backend.name)
    opt = optim.SGD(model.params(), **meta["sgd"])
    bs = batches(name, meta)
    losses = []
    for k in range(meta["steps"]):
        x, y = bs[k % 2]
        loss, _ = training.train_step(model, x, y, opt)
        losses.append(loss)
    sums = [[float(np.sum(p.numpy(), dtype=np.float64)), float(np.sum(np.abs(p.numpy()), dtype=np.float64))]
            for p in model.params()]
    return losses, sums, model
