"""Fused multi-stage reductions (pb_reduce_chain): the reference's
BatchNorm statistics x.mean(3).mean(2).mean(0) (minml/nn.py:288-306) and _unbroadcast's
sum(0).sum(2).sum(3) of a product (minml/autograd.py:290-297), traced and replayed under the
fusion plan, must equal the one-primitive-at-a-time path (same f32 roundings per stage, f64
accumulation) and the oracle's numpy f64 per-stage sums, in fewer launches."""

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
    b = GpuBackend(name="gpu-redchain", seed=1, fuse=False)
    registry.register(b)
    yield b
    registry.unregister(b.name)


def _stage(x, axis, keep, div=None):
    """One reference stage on the host: f64 sum, one f32 rounding, f32 scalar epilogue."""
    s = x.astype(np.float64).sum(axis=axis, keepdims=keep).astype(np.float32)
    return s if div is None else (s / np.float32(div)).astype(np.float32)


def _planned(be, fn):
    """fn(be) eagerly (one kernel per primitive), then traced + replayed under the plan."""
    lib = _lib.load()
    be.synchronize()
    n0 = lib.pb_launch_count()
    res = fn()
    be.synchronize()
    _planned.eager_launches = lib.pb_launch_count() - n0
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
    return eager, [t.to_host_buffer() for t in res], launches


def _ulps(a, b):
    a = np.asarray(a, np.float32).view(np.int32).astype(np.int64)
    b = np.asarray(b, np.float32).view(np.int32).astype(np.int64)
    return int(np.max(np.abs(a - b))) if a.size else 0


SHAPES = [(4, 8, 12, 12), (3, 16, 7, 7), (2, 5, 14, 14), (32, 64, 28, 28), (8, 24, 56, 56), (2, 3, 1, 9),
          (32, 2048, 7, 7)]


@pytest.mark.parametrize("shape", SHAPES)
def test_batchnorm_mean_chain(be, shape):
    r = np.random.default_rng(sum(shape))
    x = (r.standard_normal(shape) * 3 + 1).astype(np.float32)
    N, C, H, W = shape

    def fn():
        t = T.tensor(x, backend=be.name)
        c = t - t.mean(3).mean(2).mean(0).reshape((1, C, 1, 1))
        return [t.mean(3).mean(2).mean(0), (c * c).mean(3).mean(2).mean(0), t.mean(3).mean(2)]

    eager, fused, launches = _planned(be, fn)
    mu = _stage(_stage(_stage(x, 3, False, W), 2, False, H), 0, False, N)
    c = (x - mu.reshape(1, C, 1, 1)).astype(np.float32)
    var = _stage(_stage(_stage(c * c, 3, False, W), 2, False, H), 0, False, N)
    pool = _stage(_stage(x, 3, False, W), 2, False, H)
    for e, f, ref in zip(eager, fused, (mu, var, pool)):
        assert _ulps(e, f) <= 1, (shape, _ulps(e, f))
        assert _ulps(f, ref) <= 1, (shape, _ulps(f, ref))
    # chains of 2-3 stages run as one launch each (the c*c square rides in its chain); large
    # plain sources may keep their stage-at-a-time kernels (pb_reduce_chain's measured policy)
    assert launches < _planned.eager_launches, (launches, _planned.eager_launches)


@pytest.mark.parametrize("shape", SHAPES)
def test_unbroadcast_sum_chain_of_products(be, shape):
    r = np.random.default_rng(7 + sum(shape))
    g = r.standard_normal(shape).astype(np.float32)
    xh = r.standard_normal(shape).astype(np.float32)
    gam = r.standard_normal((1, shape[1], 1, 1)).astype(np.float32)

    def fn():
        tg, tx, tgam = (T.tensor(a, backend=be.name) for a in (g, xh, gam))
        def ub(t):
            return t.sum(0, keepdims=True).sum(2, keepdims=True).sum(3, keepdims=True)
        return [ub(tg), ub(tg * tx), ub(-(tg * tgam) / (tx + 4.0))]

    eager, fused, launches = _planned(be, fn)

    def ub(a):
        return _stage(_stage(_stage(a, 0, True), 2, True), 3, True)
    p2 = (g * xh).astype(np.float32)
    p3 = (-(g * gam).astype(np.float32) / (xh + np.float32(4.0)).astype(np.float32)).astype(np.float32)
    for e, f, ref in zip(eager, fused, (ub(g), ub(p2), ub(p3))):
        assert f.shape == (1, shape[1], 1, 1)
        assert _ulps(e, f) <= 1, (shape, _ulps(e, f))
        assert _ulps(f, ref) <= 1, (shape, _ulps(f, ref))
    # the products are evaluated inside the reductions
    assert launches < _planned.eager_launches - 3, (launches, _planned.eager_launches)


def test_strided_source_and_unsupported_layout_fall_back(be):
    """A transposed (non-contiguous) source and a stage order the kernel declines both give the
    one-kernel-per-stage results."""
    r = np.random.default_rng(3)
    x = r.standard_normal((6, 5, 8, 12)).astype(np.float32)

    def fn():
        t = T.tensor(x, backend=be.name).transpose((0, 1, 3, 2))  # [6, 5, 12, 8] view
        return [t.sum(3).sum(2).sum(0), t.sum(1).sum(0), (t * 2.0).sum(2).sum(0)]

    eager, fused, _ = _planned(be, fn)
    xt = x.transpose(0, 1, 3, 2)
    refs = [_stage(_stage(_stage(xt, 3, False), 2, False), 0, False), _stage(_stage(xt, 1, False), 0, False),
            _stage(_stage((xt * np.float32(2)).astype(np.float32), 2, False), 0, False)]
    for e, f, ref in zip(eager, fused, refs):
        assert _ulps(e, f) <= 1 and _ulps(f, ref) <= 1


def test_reduce_chain_abi_declines_single_stage(be):
    """pb_reduce_chain reports PB_ERR_UNSUPPORTED (nothing launched) for layouts it does not
    run, so the caller can fall back."""
    import struct
    lib = _lib.load()
    t = T.tensor(np.ones((2, 3, 4, 4), np.float32), backend=be.name)
    out = T.tensor(np.zeros((2, 3, 4), np.float32), backend=be.name)
    a, o = t.adapter, out.adapter
    n0 = lib.pb_launch_count()
    rc = lib.pb_reduce_chain(1, a.packed(), 0, 0.0, 0, b"", 4, struct.pack("<4q", 2, 3, 4, 4), 1,
                             _lib.RSTAGE.pack(3, -1, 0, 0.0), o.packed())
    assert rc == _lib.UNSUPPORTED and lib.pb_launch_count() == n0
