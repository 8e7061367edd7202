"""Throughput of all five BASELINE.json configs on one B200 (models.CONFIGS: MLP b64, LeNet
b128, AlexNet b128, ResNet-50 b32, BERT-base-like b16 seq 128), one JSON line each.

The bench contract's headline (bench.py) is ResNet-50; this is the evidence that the other
configs train on the device at full size.  Per config: `device` = steps timed with CUDA events
on the compute stream with the batch resident (CapturedStep graph replay, or eager
train_step where a graph cannot be recorded: AlexNet's dropout draws host-reserved RNG
counters every step), `e2e` = the public API with page-locked host batches (H2D + loss D2H
every step), `eager` = one Python dispatch per primitive.

    python tools/bench_configs.py [steps] [config ...]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2201_12465_b200 import models, optim, registry, training  # noqa: E402

be = registry.get("gpu")
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
names = sys.argv[2:] or list(models.CONFIGS)


def batch(cfg, r):
    b = cfg["batch"]
    if cfg.get("input") is None:
        seq, vocab = cfg["tokens"]
        x = r.integers(0, vocab, (b, seq)).astype(np.int64)
    else:
        x = r.standard_normal((b,) + tuple(cfg["input"])).astype(np.float32)
    y = r.integers(0, cfg["classes"], b).astype(np.int64)
    xp, yp = be.pinned(x.shape, x.dtype), be.pinned(y.shape, y.dtype)
    xp[...] = x
    yp[...] = y
    return xp, yp


for name in names:
    cfg = models.CONFIGS[name]
    be.seed(0)
    model = cfg["build"](be.name)
    opt = optim.SGD(model.params(), **cfg["sgd"])
    x, y = batch(cfg, np.random.default_rng(0))
    nparams = sum(int(np.prod(p.shape)) for p in model.params())
    for _ in range(2):
        training.train_step(model, x, y, opt)
    be.synchronize()
    t0 = time.perf_counter()
    stop = be.event_timer()
    n_e = 3
    for _ in range(n_e):
        training.train_step(model, x, y, opt)
    eager_ms = stop() / n_e
    step = training.CapturedStep(model, opt, warmup=2)
    mode, err = "cuda_graph", None
    try:
        for _ in range(4):
            step(x, y)
    except Exception as e:  # noqa: BLE001
        mode, err, step = "eager", f"{type(e).__name__}: {e}"[:160], None
    be.synchronize()
    stop = be.event_timer()
    if step is not None:
        for _ in range(steps):
            step.graph.launch()
    else:
        for _ in range(steps):
            training.train_step(model, x, y, opt)
    dev_ms = stop() / steps
    be.synchronize()
    stop = be.event_timer()
    if step is not None:
        losses = list(step.run([(x, y)] * steps))
    else:
        losses = [training.train_step(model, x, y, opt)[0] for _ in range(steps)]
    e2e_ms = stop() / steps
    b = cfg["batch"]
    print(json.dumps({"config": name, "batch": b, "params": nparams, "mode": mode,
                      "device": {"samples_per_s": b / dev_ms * 1e3, "ms_per_step": dev_ms},
                      "e2e": {"samples_per_s": b / e2e_ms * 1e3, "ms_per_step": e2e_ms,
                              "h2d_bytes_per_step": int(x.nbytes + y.nbytes), "d2h_bytes_per_step": 4},
                      "eager": {"samples_per_s": b / eager_ms * 1e3, "ms_per_step": eager_ms},
                      "launches_per_step": step.launches if step is not None else None,
                      "last_loss": float(losses[-1]), "graph_error": err}), flush=True)
    del model, opt, step
