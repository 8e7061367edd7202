"""Backend-internal elementwise fusion: deferred f32/bool elementwise
chains run by one pb_ew_chain launch must be bit-identical to running the same primitives
one at a time -- the GPU counterpart of the reference's eager-vs-deferred acceptance check
(T/test_acceptance.py:181-283, 200 random programs)."""

import numpy as np
import pytest

from gpu_util import gpu_backend
from paper_2201_12465_b200 import _tensor as T
from paper_2201_12465_b200 import registry
from paper_2201_12465_b200.gpu.backend import GpuBackend, LazyArray

pytestmark = pytest.mark.gpu

BIN = ["add", "sub", "mul", "div", "maximum", "minimum", "pow", "eq", "lt", "gt", "logical_and", "logical_or"]
UN = ["neg", "abs", "exp", "log", "sqrt", "tanh", "sin", "cos", "logical_not"]
SHAPES = [(4, 5, 6), (5, 1), (1, 6), (6,), (4, 1, 1), (1,)]


@pytest.fixture(scope="module")
def pair():
    gpu_backend()
    fused = GpuBackend(name="gpu-fused", seed=1, fuse=True)
    plain = GpuBackend(name="gpu-plain", seed=1, fuse=False)
    registry.register(fused)
    registry.register(plain)
    yield fused, plain
    registry.unregister(fused.name)
    registry.unregister(plain.name)


def _program(seed, be):
    """A random straight-line program over broadcastable f32/bool tensors; returns outputs."""
    r = np.random.default_rng(seed)
    pool = []
    for k in range(4):
        a = r.standard_normal(SHAPES[r.integers(len(SHAPES))]).astype(np.float32)
        if k == 3:
            a[..., 0] = np.nan if a.ndim else a
        pool.append(T.tensor(a, backend=be.name))
    pool.append(T.tensor(r.standard_normal((4, 5, 6)) > 0, backend=be.name))
    outs = []
    for _ in range(int(r.integers(3, 24))):
        op = r.choice(BIN + UN + ["astype", "scalar"])
        x = pool[int(r.integers(len(pool)))]
        if op in UN:
            try:
                y = getattr(x, op)()
            except Exception:  # noqa: BLE001 -- float-only op on a bool tensor: same on both
                continue
        elif op == "astype":
            y = x.astype("bool" if x.dtype.name == "f32" else "f32")
        elif op == "scalar":
            s = float(r.choice([0.0, 1.5, -2.0, 3]))
            if x.dtype.name == "bool":
                continue
            y = (s - x) if r.integers(2) else (x * s)
        else:
            z = pool[int(r.integers(len(pool)))]
            if op in ("pow",) and (x.dtype.name == "bool" or z.dtype.name == "bool"):
                continue
            try:
                y = getattr(x, op)(z)
            except Exception:  # noqa: BLE001 -- same planning error on both backends
                continue
        pool.append(y)
        if r.integers(3) == 0:
            outs.append(y)
    outs.append(pool[-1])
    return [o.to_host_buffer() for o in outs]


@pytest.mark.parametrize("seed", range(200))
def test_random_programs_fused_equal_unfused(pair, seed):
    fused, plain = pair
    with np.errstate(all="ignore"):
        got = _program(seed, fused)
        want = _program(seed, plain)
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert g.dtype == w.dtype and g.shape == w.shape
        assert np.array_equal(g, w, equal_nan=True), (seed, g, w)


def test_chains_defer_and_materialise_once(pair):
    fused, _ = pair
    r = np.random.default_rng(0)
    x = T.tensor(r.standard_normal((32, 64, 8, 8)).astype(np.float32), backend=fused.name)
    mu = T.tensor(r.standard_normal((1, 64, 1, 1)).astype(np.float32), backend=fused.name)
    sd = T.tensor(r.random((1, 64, 1, 1)).astype(np.float32) + 0.5, backend=fused.name)
    n0 = fused.launch_count()
    y = (((x - mu) / sd) * 2.0 + 0.5).maximum(0)     # BatchNorm-affine + ReLU: one chain
    mask = y.lt(0).logical_not().astype("f32")       # ReLU mask: extends y's chain
    assert type(y.adapter) is LazyArray and type(mask.adapter) is LazyArray
    assert fused.launch_count() == n0                # nothing launched yet
    out = (mask * y).sum()                           # the reduction forces one fused launch
    assert fused.launch_count() - n0 <= 4
    xs = x.numpy()
    want = np.maximum(((xs - mu.numpy()) / sd.numpy()) * np.float32(2.0) + np.float32(0.5), 0)
    assert np.array_equal(y.numpy(), want)
    assert np.isfinite(out.scalar())


def test_lazy_results_feed_views_and_contractions(pair):
    fused, plain = pair
    r = np.random.default_rng(1)
    a = r.standard_normal((16, 24)).astype(np.float32)
    b = r.standard_normal((24, 8)).astype(np.float32)
    res = []
    for be in (fused, plain):
        ta, tb = T.tensor(a, backend=be.name), T.tensor(b, backend=be.name)
        h = (ta * 2.0).tanh()
        res.append([(h @ tb).numpy(), h.transpose().numpy(), h.reshape((4, 96)).numpy(),
                    h.slice((0, 0), (16, 24), (2, 3)).numpy(), h.sum(axis=1).numpy()])
    for g, w in zip(*res):
        assert np.array_equal(g, w)


def test_chain_kernels_are_jit_specialised(pair):
    """The fused chains above ran as NVRTC-specialised kernels (pb_chain_jit_kernels), not only
    through the interpreter; their results were already compared bit for bit with the unfused
    primitives."""
    from paper_2201_12465_b200.gpu import _lib
    n = _lib.load().pb_chain_jit_kernels()
    assert n > 0, n
