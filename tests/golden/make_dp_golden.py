"""Data-parallel golden fixtures from the REFERENCE's own thread-rank runs (minml
distributed.run_ranks + training.train_step(comm=...)), made in the build container.

    PB_NO_AUTOREGISTER=1 python tests/golden/make_dp_golden.py

1. ``acceptance``: the reference's acceptance fixture T/test_acceptance.py:394-440 -- MLP
   784-128-10, SGD lr 0.05, data.synth_blobs(320, seed=21, dim=784) in global batches of 32,
   50 steps; 4 ranks x 8 vs 1 rank x 32.  Records the single-rank losses, every rank's
   losses and the final parameter sums of rank 0.  The 320 host samples are stored too
   (the synth_blobs generator is the reference's data subsystem, out of scope here).
2. ``bn``: SURVEY §8(e3) -- BatchNorm keeps per-rank batch statistics, so a DP ResNet run
   equals the reference's thread-rank run on the same shards, not a single-rank run.  A
   reduced ResNet (layers 1-1-1-1, width 8) on 2 ranks x 4 samples, SGD(0.05, momentum
   0.9), 4 steps: per-rank losses, parameter sums, and BN running statistics of rank 0.

Outputs (committed): dp.json, dp.npz.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
os.environ.setdefault("PB_NO_AUTOREGISTER", "1")

from minml import _tensor as MT, autograd as MA, data as MD, distributed as MDist  # noqa: E402
from minml import models as MMod, nn as MN, ops as MO, optim as MOpt, registry as MR  # noqa: E402
from minml import training as MTr  # noqa: E402
from minml.eager import EagerBackend  # noqa: E402

from paper_2201_12465_b200 import models as PM  # noqa: E402

sys.path.insert(0, HERE)
import inputs as GI  # noqa: E402

NS = PM.namespace(MN, MO, MT, MA)


def acceptance():
    world, per_rank, steps = 4, 8, 50
    ds = MD.synth_blobs(320, seed=21, dim=784)
    batches = MD.Batch(ds, world * per_rank, drop_last=True)
    host = [batches[k] for k in range(len(batches))]

    def build(name):
        MR.register(EagerBackend(name=name, seed=13))
        model = MMod.mlp(784, 128, 10, backend=name)
        return model, MOpt.SGD(model.params(), lr=0.05)

    single = []
    model, opt = build("g-dp-single")
    try:
        for k in range(steps):
            images, labels = host[k % len(host)]
            single.append(float(MTr.train_step(model, images, labels, opt)[0]))
    finally:
        MR.unregister("g-dp-single")

    def fn(comm):
        model = MMod.mlp(784, 128, 10, backend=f"g-dp-{comm.rank}")
        opt = MOpt.SGD(model.params(), lr=0.05)
        losses, lo = [], comm.rank * per_rank
        for k in range(steps):
            images, labels = host[k % len(host)]
            losses.append(float(MTr.train_step(model, images[lo:lo + per_rank], labels[lo:lo + per_rank], opt,
                                               comm=comm)[0]))
        sums = [float(np.sum(p.numpy(), dtype=np.float64)) for p in model.params()]
        return losses, sums

    for r in range(world):
        MR.register(EagerBackend(name=f"g-dp-{r}", seed=13))
    try:
        res = MDist.run_ranks(world, fn)
    finally:
        for r in range(world):
            MR.unregister(f"g-dp-{r}")
    images = np.concatenate([b[0] for b in host])
    labels = np.concatenate([b[1] for b in host])
    meta = {"world": world, "per_rank": per_rank, "steps": steps, "seed": 13, "lr": 0.05,
            "single": single, "ranks": [r[0] for r in res], "param_sums": res[0][1],
            "n_batches": len(host)}
    return meta, {"acc_images": images.astype(np.float32), "acc_labels": labels.astype(np.int64)}


def bn():
    world, per, steps = 2, 4, 4
    bs = [GI.batch("dp_bn", k, (3, 32, 32), 10, world * per) for k in range(2)]

    def fn(comm):
        model = PM.resnet50(classes=10, layers=(1, 1, 1, 1), width=8, backend=f"g-bn-{comm.rank}", ns=NS)
        opt = MOpt.SGD(model.params(), lr=0.05, momentum=0.9)
        losses = []
        for k in range(steps):
            x, y = bs[k % 2]
            lo = comm.rank * per
            losses.append(float(MTr.train_step(model, x[lo:lo + per], y[lo:lo + per], opt, comm=comm)[0]))
        sums = [float(np.sum(p.numpy(), dtype=np.float64)) for p in model.params()]
        stats = []

        def walk(m):
            for name in m.buffer_names():
                stats.append(float(np.sum(getattr(m, name).numpy(), dtype=np.float64)))
            for _, c in m._children:
                walk(c)
        walk(model)
        return losses, sums, stats

    for r in range(world):
        MR.register(EagerBackend(name=f"g-bn-{r}", seed=17))
    try:
        res = MDist.run_ranks(world, fn)
    finally:
        for r in range(world):
            MR.unregister(f"g-bn-{r}")
    return {"world": world, "per_rank": per, "steps": steps, "seed": 17, "ranks": [r[0] for r in res],
            "param_sums": [r[1] for r in res], "buffer_sums": [r[2] for r in res]}


def main():
    acc, arrays = acceptance()
    meta = {"acceptance": acc, "bn": bn()}
    gap = max(abs(float(np.mean([acc["ranks"][r][k] for r in range(acc["world"])])) - acc["single"][k])
              for k in range(acc["steps"]))
    print(f"acceptance: worst mean-vs-single gap {gap:.2e}; bn ranks {meta['bn']['ranks']}")
    with open(os.path.join(HERE, "dp.json"), "w") as f:
        json.dump(meta, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "dp.npz"), **arrays)


if __name__ == "__main__":
    main()
