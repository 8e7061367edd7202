"""Whole-step CUDA graph replay (training.CapturedStep) against the eager
``train_step`` (minml/training.py:37-51): the same kernels on the same buffers, so losses,
parameters, momentum buffers and BatchNorm running statistics must be bit-identical."""

import numpy as np
import pytest

from frontend_util import BUILDERS
from gpu_util import gpu_backend
from paper_2201_12465_b200 import models, optim, training

pytestmark = pytest.mark.gpu


def _run(name, be, captured, steps, batch, shape, classes, seed=3, fuse=False):
    be.seed(seed)
    model = BUILDERS[name](be.name)
    opt = optim.SGD(model.params(), lr=0.05, momentum=0.9)
    r = np.random.default_rng(0)
    data = [(r.standard_normal((batch,) + shape).astype(np.float32), r.integers(0, classes, batch).astype(np.int64))
            for _ in range(2)]
    step = (training.CapturedStep(model, opt, warmup=2 if fuse else 1, fuse=fuse) if captured else None)
    losses = []
    for k in range(steps):
        x, y = data[k % 2]
        if captured:
            loss, _ = step(x, y)
        else:
            loss, _ = training.train_step(model, x, y, opt)
        losses.append(loss)
    params = [p.numpy() for p in model.params()]
    vel = [v.numpy() for v in opt.velocity]
    bufs = []

    def walk(m):
        for nme in m.buffer_names():
            bufs.append(getattr(m, nme).numpy())
        for _, c in m._children:
            walk(c)
    walk(model)
    return losses, params, vel, bufs, step


@pytest.mark.parametrize("name,shape,classes", [("lenet", (1, 28, 28), 10), ("resnet_tiny", (3, 32, 32), 10)])
def test_captured_step_bit_identical_to_eager(name, shape, classes):
    be = gpu_backend()
    eager = _run(name, be, False, 6, 4, shape, classes)
    graph = _run(name, be, True, 6, 4, shape, classes)
    step = graph[4]
    assert step.graph is not None and step.launches > 20
    assert eager[0] == graph[0], (eager[0], graph[0])
    for a, b in zip(eager[1] + eager[2] + eager[3], graph[1] + graph[2] + graph[3]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("name,shape,classes", [("lenet", (1, 28, 28), 10), ("resnet_tiny", (3, 32, 32), 10)])
def test_planned_fusion_bit_identical_and_fewer_launches(name, shape, classes):
    """The traced-then-planned fusion (GpuBackend.fusion_*) folds single-consumer elementwise
    results into chain kernels: fewer launches, bit-identical losses and state."""
    be = gpu_backend()
    eager = _run(name, be, False, 6, 4, shape, classes)
    plain = _run(name, be, True, 6, 4, shape, classes)
    fused = _run(name, be, True, 6, 4, shape, classes, fuse=True)
    step = fused[4]
    assert step.fused_ops > 0 and step.launches < plain[4].launches, (step.fused_ops, step.launches,
                                                                     plain[4].launches)
    assert step.plan_abandoned is False  # the recorded step followed its trace to the end
    assert eager[0] == fused[0], (eager[0], fused[0])
    for a, b in zip(eager[1] + eager[2] + eager[3], fused[1] + fused[2] + fused[3]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("name,shape,classes", [("lenet", (1, 28, 28), 10), ("resnet_tiny", (3, 32, 32), 10)])
def test_chain_taps_bit_identical_and_fewer_launches(name, shape, classes, monkeypatch):
    """Taps (pb_ew_chain_taps): a multi-use elementwise intermediate -- BatchNorm's xhat, the
    affine output before the ReLU -- is stored by its first consumer's chain kernel instead of
    a pass of its own.  Same losses and state bit for bit, fewer launches than without taps."""
    from paper_2201_12465_b200.gpu import backend as gb
    be = gpu_backend()
    monkeypatch.setattr(gb, "_TAPS", False)
    off = _run(name, be, True, 6, 4, shape, classes, fuse=True)
    monkeypatch.setattr(gb, "_TAPS", True)
    on = _run(name, be, True, 6, 4, shape, classes, fuse=True)
    assert on[4].plan_abandoned is False
    if name == "resnet_tiny":  # (LeNet has no BatchNorm chains to tap)
        assert on[4].launches < off[4].launches, (on[4].launches, off[4].launches)
    assert on[4].launches <= off[4].launches
    assert on[0] == off[0], (on[0], off[0])
    for a, b in zip(off[1] + off[2] + off[3], on[1] + on[2] + on[3]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("fuse", [False, True])
def test_captured_dropout_draws_fresh_masks_bit_identical(fuse):
    """Dropout (minml/nn.py:247-256) inside the graph: each replay draws the counter range the
    host reserves for it (pb_rand_dev + GraphExec), so the masks, losses, parameters and the
    host RNG counter equal those of the same number of eager steps."""
    be = gpu_backend()
    eager = _run("alexnet_tiny", be, False, 6, 4, (3, 67, 67), 10)
    eager_next = be.rng.state()["next"]
    graph = _run("alexnet_tiny", be, True, 6, 4, (3, 67, 67), 10, fuse=fuse)
    assert graph[4].graph is not None and graph[4].graph.rng_per_step > 0
    assert be.rng.state()["next"] == eager_next
    assert eager[0] == graph[0], (eager[0], graph[0])
    for a, b in zip(eager[1] + eager[2], graph[1] + graph[2]):
        assert np.array_equal(a, b)


def test_captured_dropout_follows_foreign_reservations():
    """An eager random draw between replays moves the host counter; the next replay rewrites
    the device counter and still draws exactly what the eager step would."""
    from paper_2201_12465_b200 import _tensor as T
    be = gpu_backend()
    runs = []
    for captured in (False, True):
        be.seed(9)
        model = BUILDERS["alexnet_tiny"](be.name)
        opt = optim.SGD(model.params(), lr=0.01)
        r = np.random.default_rng(1)
        x = r.standard_normal((2, 3, 67, 67)).astype(np.float32)
        y = r.integers(0, 10, 2).astype(np.int64)
        step = training.CapturedStep(model, opt, warmup=1, fuse=False) if captured else None
        losses = []
        for k in range(5):
            if k == 3:
                T.rand_uniform((7,), backend=be.name)  # a foreign reservation
            losses.append(step(x, y)[0] if captured else training.train_step(model, x, y, opt)[0])
        runs.append((losses, [p.numpy() for p in model.params()]))
    assert runs[0][0] == runs[1][0]
    for a, b in zip(runs[0][1], runs[1][1]):
        assert np.array_equal(a, b)


def test_captured_step_checks_targets():
    be = gpu_backend()
    be.seed(1)
    lenet = models.mnist_cnn(backend=be.name)
    st = training.CapturedStep(lenet, optim.SGD(lenet.params(), lr=0.01), warmup=1)
    xs = np.zeros((2, 1, 28, 28), np.float32)
    st(xs, np.zeros(2, np.int64))
    st(xs, np.zeros(2, np.int64))
    with pytest.raises(IndexError):
        st(xs, np.array([0, 10], np.int64))


@pytest.mark.parametrize("name,shape,classes", [("lenet", (1, 28, 28), 10), ("resnet_tiny", (3, 32, 32), 10)])
def test_pipelined_run_bit_identical_to_eager(name, shape, classes):
    """CapturedStep.run (copy-stream H2D of batch i+1 under step i, posted loss reads) yields
    the eager train_step losses in order and leaves bit-identical state; 7 steps cross the
    two staging slots and the eight read slots."""
    be = gpu_backend()
    eager = _run(name, be, False, 7, 4, shape, classes)
    be.seed(3)
    model = BUILDERS[name](be.name)
    opt = optim.SGD(model.params(), lr=0.05, momentum=0.9)
    r = np.random.default_rng(0)
    data = [(r.standard_normal((4,) + shape).astype(np.float32), r.integers(0, classes, 4).astype(np.int64))
            for _ in range(2)]
    step = training.CapturedStep(model, opt, warmup=1, fuse=False)
    losses = list(step.run(data[k % 2] for k in range(7)))
    assert step.graph is not None
    assert losses == eager[0], (losses, eager[0])
    for a, b in zip(eager[1], [p.numpy() for p in model.params()]):
        assert np.array_equal(a, b)


def test_pipelined_run_checks_targets():
    be = gpu_backend()
    be.seed(3)
    model = BUILDERS["lenet"](be.name)
    opt = optim.SGD(model.params(), lr=0.05)
    x = np.zeros((4, 1, 28, 28), np.float32)
    good, bad = np.array([0, 1, 2, 3]), np.array([0, 1, 2, 10])
    step = training.CapturedStep(model, opt, warmup=1, fuse=False)
    with pytest.raises(IndexError):
        list(step.run([(x, good), (x, good), (x, bad)]))


def test_pinned_batches_match_pageable():
    """Batches in page-locked memory (one DMA, no staging copy) give the same losses."""
    be = gpu_backend()
    losses = []
    for pin in (False, True):
        be.seed(3)
        model = BUILDERS["lenet"](be.name)
        opt = optim.SGD(model.params(), lr=0.05, momentum=0.9)
        r = np.random.default_rng(0)
        x = r.standard_normal((4, 1, 28, 28)).astype(np.float32)
        y = r.integers(0, 10, 4).astype(np.int64)
        if pin:
            xp, yp = be.pinned(x.shape, x.dtype), be.pinned(y.shape, y.dtype)
            xp[...] = x
            yp[...] = y
            x, y = xp, yp
        step = training.CapturedStep(model, opt, warmup=1, fuse=False)
        losses.append(list(step.run([(x, y)] * 5)))
    assert losses[0] == losses[1]
