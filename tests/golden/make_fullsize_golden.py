"""Full-size golden trajectories: the five BASELINE.json configs at their real width and
depth, run by the REFERENCE (minml's EagerBackend) in the build container.

    PB_NO_AUTOREGISTER=1 python tests/golden/make_fullsize_golden.py [name ...]

Needs /root/reference (read-only); it runs only here, never on the GPU box.  Each config
trains for 10 steps (minml/training.py:37-51 train_step, alternating two synthetic batches
from tests/golden/inputs.py) and records, per step, the loss, and at the end, per parameter
tensor: sum, sum|p|, and 64 elements at fixed sampled flat indices.  Each config is also
run from an init perturbed by 1e-7 (relative): the loss gap of that run is the reference's
own conditioning ("self_sensitivity", ~what one ulp of f32 noise does).  ResNet-50 is the
ill-conditioned one: a 1e-7 perturbation moves its 10-step losses by 7e-2 at batch 2 / lr
1e-3, 1.7e-2 at batch 2 / lr 1e-5 and 7e-3 at batch 8 / lr 1e-4 (the recorded config); the
perturbed run's parameter gaps are recorded too ("self_sensitivity_params").  MLP and LeNet run at
their BASELINE batch (64, 128); AlexNet, ResNet-50 and BERT-base at batch 2 (the reference's
numpy step at batch 32 takes about a minute).  Compositions come from
paper_2201_12465_b200.models bound to minml's own nn/ops/_tensor/autograd, so both sides
run the identical primitive stream.

Outputs (committed): fullsize.json, fullsize.npz.
"""

import json
import os
import sys
import time

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
STEPS = 10
SAMPLES = 64

# name -> (builder(backend, ns), input shape or None for tokens, classes, batch, sgd, tokens)
CONFIGS = {
    "mlp_full": (lambda be, ns: PM.mlp(784, 256, 10, backend=be, ns=ns), (784,), 10, 64,
                 dict(lr=0.05), None),
    "lenet_full": (lambda be, ns: PM.mnist_cnn(backend=be, ns=ns), (1, 28, 28), 10, 128,
                   dict(lr=0.05, momentum=0.9), None),
    "alexnet_full": (lambda be, ns: PM.alexnet(backend=be, ns=ns), (3, 224, 224), 1000, 2,
                     dict(lr=0.01, momentum=0.9), None),
    "resnet50_full": (lambda be, ns: PM.resnet50(backend=be, ns=ns), (3, 224, 224), 1000, 8,
                      dict(lr=1e-4, momentum=0.9), None),
    "bert_full": (lambda be, ns: PM.bert_base(backend=be, ns=ns), None, 2, 2,
                  dict(lr=0.001, momentum=0.9), (128, 30522)),
}


def sample_index(name, i, size):
    r = np.random.default_rng(7919 * i + len(name))
    return np.sort(r.choice(size, size=min(SAMPLES, size), replace=False))


def batches(name):
    _, shape, classes, batch, _, tokens = CONFIGS[name]
    return [GI.batch(name, k, shape, classes, batch, tokens=tokens) for k in range(2)]


def run(name, perturb=0.0):
    build, _, _, _, sgd, _ = CONFIGS[name]
    be_name = f"full-{name}"
    MR.register(EagerBackend(name=be_name, seed=5))
    t0 = time.perf_counter()
    try:
        model = build(be_name, NS)
        if perturb:  # conditioning probe: every parameter scaled by (1 + perturb * N(0,1))
            r = np.random.default_rng(1)
            for p in model.params():
                a = p.numpy()
                p.data = MT.tensor((a * (1 + perturb * r.standard_normal(a.shape))).astype(np.float32),
                                   backend=be_name)
        opt = MOpt.SGD(model.params(), **sgd)
        bs = batches(name)
        losses = []
        for k in range(STEPS):
            x, y = bs[k % 2]
            loss, _ = MTr.train_step(model, x, y, opt)
            losses.append(float(loss))
        params = [p.numpy() for p in model.params()]
    finally:
        MR.unregister(be_name)
    sums = [[float(np.sum(p, dtype=np.float64)), float(np.sum(np.abs(p), dtype=np.float64))] for p in params]
    arrays = {}
    for i, p in enumerate(params):
        idx = sample_index(name, i, p.size)
        arrays[f"{name}_p{i}_idx"] = idx.astype(np.int64)
        arrays[f"{name}_p{i}_val"] = p.reshape(-1)[idx]
    meta = {"losses": losses, "param_sums": sums, "seed": 5, "steps": STEPS, "sgd": sgd,
            "n_params": len(params), "shapes": [list(p.shape) for p in params],
            "batch": CONFIGS[name][3], "ref_seconds": time.perf_counter() - t0}
    return meta, arrays


def main():
    names = sys.argv[1:] or list(CONFIGS)
    jpath, npath = os.path.join(HERE, "fullsize.json"), os.path.join(HERE, "fullsize.npz")
    meta = json.load(open(jpath)) if os.path.exists(jpath) else {}
    arrays = dict(np.load(npath)) if os.path.exists(npath) else {}
    for name in names:
        m, a = run(name)
        # the reference's own conditioning: the same run from an init perturbed by 1e-7
        # (relative), i.e. what ~1 ulp of f32 noise does to the 10-step trajectory
        mp, ap = run(name, perturb=1e-7)
        rel = lambda u, v: abs(u - v) / max(abs(u), abs(v), 1.0)  # noqa: E731
        m["self_sensitivity"] = max(rel(u, v) for u, v in zip(m["losses"], mp["losses"]))
        m["self_sensitivity_params"] = {
            "sum": max(rel(u[0], v[0]) for u, v in zip(m["param_sums"], mp["param_sums"])),
            "abs_sum": max(rel(u[1], v[1]) for u, v in zip(m["param_sums"], mp["param_sums"])),
            "sampled": max(float(np.max(np.abs(a[k] - ap[k]) / np.maximum(np.maximum(np.abs(a[k]), np.abs(ap[k])), 1)))
                           for k in a if k.endswith("_val"))}
        meta[name] = m
        arrays = {k: v for k, v in arrays.items() if not k.startswith(name + "_")}
        arrays.update(a)
        print(f"{name}: {m['ref_seconds']:.1f} s, losses {m['losses'][0]:.5f} .. {m['losses'][-1]:.5f}, "
              f"self-sensitivity {m['self_sensitivity']:.1e}", flush=True)
        with open(jpath, "w") as f:
            json.dump(meta, f, indent=1)
        np.savez_compressed(npath, **arrays)


if __name__ == "__main__":
    main()
