"""Windowed chain leaves (LazyWindow / pb_ew_chain_win): under the fusion plan a
pad, a zero-stuffing pad + reshape, or a strided slice of a padded tensor is not materialised;
the chain kernel reads the source through the window.  Values must equal the eager primitives
bit for bit: the maxpool forward's -inf pad and 9 strided windows (minml/nn.py MaxPool2d) and the
slice backward's zero-stuffing scatter (minml/autograd.py:667-693)."""

import numpy as np
import pytest

from gpu_util import gpu_backend
from paper_2201_12465_b200 import _tensor as T
from paper_2201_12465_b200 import registry
from paper_2201_12465_b200.gpu import _lib
from paper_2201_12465_b200.gpu.backend import GpuBackend

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def be():
    gpu_backend()
    b = GpuBackend(name="gpu-window", seed=1, fuse=False)
    registry.register(b)
    yield b
    registry.unregister(b.name)


def _planned(be, fn):
    lib = _lib.load()
    be.synchronize()
    n0 = lib.pb_launch_count()
    res = fn()
    be.synchronize()
    eager_launches = lib.pb_launch_count() - n0
    eager = [t.to_host_buffer() for t in res]
    be.fusion_trace_begin()
    fn()
    be.fusion_trace_end()
    be.synchronize()
    n0 = lib.pb_launch_count()
    assert be.fusion_plan_begin()
    try:
        res = fn()
        abandoned = be.plan_abandoned
    finally:
        be.fusion_plan_end()
    be.synchronize()
    launches = lib.pb_launch_count() - n0
    assert not abandoned
    return eager, [t.to_host_buffer() for t in res], eager_launches, launches


def _same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("shape", [(2, 3, 9, 9), (4, 8, 16, 16), (32, 64, 28, 28), (3, 5, 7, 12)])
def test_maxpool_windows_forward(be, shape):
    """pad(-inf) then the 9 stride-2 windows folded with maximum, as the reference's maxpool."""
    x = np.random.default_rng(1).standard_normal(shape).astype(np.float32)
    N, C, H, W = shape

    def fn():
        t = T.tensor(x, backend=be.name).pad(((0, 0), (0, 0), (1, 1), (1, 1)), value=float("-inf"))
        ho, wo = (H + 2 - 3) // 2 + 1, (W + 2 - 3) // 2 + 1
        m = None
        for r in range(3):
            for s in range(3):
                win = t.slice((0, 0, r, s), (N, C, r + 2 * (ho - 1) + 1, s + 2 * (wo - 1) + 1), (1, 1, 2, 2))
                m = win if m is None else m.maximum(win)
        return [m, m.lt(0.5)]

    eager, fused, n_e, n_f = _planned(be, fn)
    for e, f in zip(eager, fused):
        assert _same(e, f)
    assert n_f < n_e, (n_f, n_e)


@pytest.mark.parametrize("shape", [(2, 3, 5, 5), (4, 8, 14, 14), (32, 64, 28, 28)])
def test_zero_stuffing_scatter_sum(be, shape):
    """The slice backward's scatter (reshape, pad, reshape, slice, pad per strided axis) of
    several window grads, summed -- the maxpool backward's pattern."""
    rng = np.random.default_rng(2)
    N, C, H, W = shape
    Hp, Wp = 2 * H + 2, 2 * W + 2
    gs = [rng.standard_normal(shape).astype(np.float32) for _ in range(4)]
    starts = [(0, 0), (0, 1), (1, 0), (1, 1)]

    def scatter(t, r0, s0):
        for ax, (start, dim) in ((2, (r0, Hp)), (3, (s0, Wp))):
            s = tuple(t.shape)
            m = s[ax]
            t = t.reshape(s[:ax] + (m, 1) + s[ax + 1:])
            pads = [(0, 0)] * (len(s) + 1)
            pads[ax + 1] = (0, 1)
            t = t.pad(pads).reshape(s[:ax] + (2 * m,) + s[ax + 1:])
            covered = 2 * (m - 1) + 1
            hi = list(t.shape)
            hi[ax] = covered
            t = t.slice([0] * len(s), hi)
            pads = [(0, 0)] * len(s)
            pads[ax] = (start, dim - start - covered)
            t = t.pad(pads)
        return t

    def fn():
        acc = None
        for g, (r0, s0) in zip(gs, starts):
            c = scatter(T.tensor(g, backend=be.name), r0, s0)
            acc = c if acc is None else acc + c
        return [acc, acc * 2.0]

    eager, fused, n_e, n_f = _planned(be, fn)
    for e, f in zip(eager, fused):
        assert _same(e, f)
    assert n_f < n_e, (n_f, n_e)


def test_window_materialises_for_other_consumers(be):
    """A windowed tensor that meets a non-elementwise consumer is materialised with the eager
    pad's values (fill + strided copy, or the chain kernel for strided windows)."""
    x = np.random.default_rng(3).standard_normal((2, 3, 6, 6)).astype(np.float32)

    def fn():
        t = T.tensor(x, backend=be.name)
        p = t.pad(((0, 0), (0, 0), (2, 1), (0, 3)), value=1.5)
        s = p.slice((0, 0, 1, 0), (2, 3, 9, 9), (1, 1, 2, 3))
        return [p.sum(3), s.transpose((0, 1, 3, 2)).reshape((2, 3, 12)), p.reshape((2, 3, 81))]

    eager, fused, _, _ = _planned(be, fn)
    for e, f in zip(eager, fused):
        assert _same(e, f)
