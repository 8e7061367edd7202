"""Per-primitive parity of the CUDA backend against the reference's own outputs
(tests/golden/ops.*) and against the numpy oracle on strided views and large sizes.

Tolerances: bit-exact for integer / bool / index / movement / creation results and for
IEEE-exact f32 ops (+ - * / sqrt, min/max, compares); rel 1e-5 (|a-b|/max(|a|,|b|,1),
the reference's metric) for transcendental ops, reductions and contractions."""

import numpy as np
import pytest

from golden_util import assert_contraction, check_against, f32_conv_family, op_cases, rel_err
from gpu_util import gpu_backend
from paper_2201_12465_b200 import _tensor as T
from paper_2201_12465_b200 import errors

pytestmark = pytest.mark.gpu
CASES = op_cases()


@pytest.fixture(scope="module")
def gpu():
    return gpu_backend()


@pytest.mark.parametrize("case", CASES, ids=[c["id"] for c in CASES])
def test_golden_case(case, gpu):
    ins = [T.tensor(a, backend=gpu.name) for a in case["input_arrays"]]
    if "error" in case:
        with pytest.raises((errors.Error, ValueError, OverflowError)) as ei:
            out = T.apply(case["name"], case["params"], ins, backend=None if ins else gpu)
            out.to_host_buffer()
        assert type(ei.value).__name__ == case["error"]
        return
    out = T.apply(case["name"], case["params"], ins, backend=None if ins else gpu)
    got = out.to_host_buffer()
    tol = 1e-5
    if case["name"] == "rand_normal":
        tol = 1e-6
    check_against(case, got, tol=tol)


def _oracle(name, params, arrays):
    from oracle.kernels import KERNELS
    from paper_2201_12465_b200 import dtypes, infer
    from paper_2201_12465_b200.registry import OpCall
    from paper_2201_12465_b200.shape import Shape
    ins = [(Shape(a.shape), dtypes.from_numpy(a.dtype)) for a in arrays]
    shape, dt = infer.plan(name, params, ins)
    return KERNELS[name](OpCall(name, params, shape, dt), arrays)


def test_views_feed_every_kernel(gpu):
    r = np.random.default_rng(1)
    a = r.standard_normal((6, 5, 7)).astype(np.float32)
    b = r.standard_normal((7, 5)).astype(np.float32)
    ta, tb = T.tensor(a, backend=gpu.name), T.tensor(b, backend=gpu.name)
    at = ta.transpose((2, 1, 0))            # [7,5,6] strided view
    sl = ta.slice((1, 0, 2), (6, 5, 7), (2, 2, 1))
    # binary on views with broadcasting
    got = (at * tb.reshape((7, 5, 1))).to_host_buffer()
    assert np.array_equal(got, np.transpose(a, (2, 1, 0)) * b.reshape(7, 5, 1))
    assert np.array_equal(sl.exp().to_host_buffer(), np.exp(a[1:6:2, 0:5:2, 2:7]) ) or \
        rel_err(sl.exp().to_host_buffer(), np.exp(a[1:6:2, 0:5:2, 2:7])) < 1e-6
    # reductions over strided axes
    for ax in (0, 1, 2):
        want = np.sum(np.transpose(a, (2, 1, 0)), axis=ax, dtype=np.float64).astype(np.float32)
        assert rel_err(at.sum(axis=ax).to_host_buffer(), want) < 1e-6
        assert np.array_equal(at.argmax(ax).to_host_buffer(), np.argmax(np.transpose(a, (2, 1, 0)), axis=ax))
    # matmul with transposed operands (Linear's W^T, matmul backward)
    w = r.standard_normal((9, 5)).astype(np.float32)
    x = r.standard_normal((4, 5)).astype(np.float32)
    tw, tx = T.tensor(w, backend=gpu.name), T.tensor(x, backend=gpu.name)
    want = (x.astype(np.float64) @ w.T.astype(np.float64)).astype(np.float32)
    assert rel_err((tx @ tw.transpose()).to_host_buffer(), want) < 1e-5
    want = (x.T.astype(np.float64) @ x.astype(np.float64)).astype(np.float32)
    assert rel_err((tx.transpose() @ tx).to_host_buffer(), want) < 1e-5
    # full() is a stride-0 view; consumers and to_host see the dense value
    f = T.full((3, 4), 2.5, backend=gpu.name)
    assert np.array_equal(f.to_host_buffer(), np.full((3, 4), 2.5, np.float32))
    assert np.array_equal((f * tb.slice((0, 0), (3, 4))).to_host_buffer(), 2.5 * b[:3, :4])
    # concat of views, pad of a view
    c = T.concat([at.slice((0, 0, 0), (7, 5, 2)), tb.reshape((7, 5, 1))], 2).to_host_buffer()
    assert np.array_equal(c, np.concatenate([np.transpose(a, (2, 1, 0))[:, :, :2], b.reshape(7, 5, 1)], 2))
    p = at.pad(((1, 0), (0, 2), (3, 1)), value=-1.5).to_host_buffer()
    assert np.array_equal(p, np.pad(np.transpose(a, (2, 1, 0)), ((1, 0), (0, 2), (3, 1)), constant_values=-1.5))


@pytest.mark.parametrize("n", [1, 7, 4096 * 4096 + 13])
def test_large_sum_f64_accumulation(gpu, n):
    x = np.random.default_rng(n % 1000).standard_normal(n).astype(np.float32) * 100
    got = T.tensor(x, backend=gpu.name).sum().to_host_buffer()
    want = np.sum(x, dtype=np.float64).astype(np.float32)
    assert rel_err(got, want) <= 1e-6


def test_large_elementwise_bit_exact(gpu):
    r = np.random.default_rng(3)
    a = r.standard_normal(1 << 24).astype(np.float32)
    b = r.standard_normal(1 << 24).astype(np.float32)
    ta, tb = T.tensor(a, backend=gpu.name), T.tensor(b, backend=gpu.name)
    for op, f in (("add", np.add), ("mul", np.multiply), ("div", np.divide), ("maximum", np.maximum)):
        assert np.array_equal(getattr(ta, op)(tb).to_host_buffer(), f(a, b))
    assert np.array_equal(ta.lt(0).logical_not().astype("f32").to_host_buffer(),
                          np.logical_not(a < 0).astype(np.float32))


PADS = [
    ((4, 8, 14, 1, 14), ((0, 0), (0, 0), (0, 0), (0, 1), (0, 0)), 0.0),   # max-pool backward interleave
    ((4, 8, 27, 28), ((0, 0), (0, 0), (1, 0), (0, 0)), 0.0),             # rows, inner extent % 4 == 0
    ((4, 8, 28, 27), ((0, 0), (0, 0), (0, 0), (2, 1)), 0.0),             # inner offset not 16B aligned
    ((2, 3, 7, 7), ((0, 0), (0, 0), (1, 1), (1, 1)), float("-inf")),    # stem pad before max-pool
    ((5, 6, 3), ((2, 1), (0, 0), (1, 0)), -2.5),
]


@pytest.mark.parametrize("shape,pw,value", PADS)
def test_pad_layouts(gpu, shape, pw, value):
    x = np.random.default_rng(len(shape)).standard_normal(shape).astype(np.float32)
    t = T.tensor(x, backend=gpu.name)
    assert np.array_equal(t.pad(pw, value=value).to_host_buffer(), np.pad(x, pw, constant_values=value))
    # strided source view (transposed last two axes)
    perm = tuple(range(len(shape) - 2)) + (len(shape) - 1, len(shape) - 2)
    xv = np.transpose(x, perm)
    pv = pw[:-2] + (pw[-1], pw[-2])
    assert np.array_equal(t.transpose(perm).pad(pv, value=value).to_host_buffer(),
                          np.pad(xv, pv, constant_values=value))


@pytest.mark.parametrize("shape,axis", [((32, 64, 56, 56), 3), ((32, 64, 56), 2), ((32, 2048), 0), ((2048, 768), 0),
                                        ((16, 1000), 1), ((3, 100003), 1), ((32, 64, 7, 7), 3), ((32, 64, 28), 2),
                                        ((1, 64, 14, 14), 2), ((32, 64, 5), 0), ((2, 3, 33), 2)])
def test_reduction_shapes(gpu, shape, axis):
    x = np.random.default_rng(7).standard_normal(shape).astype(np.float32)
    t = T.tensor(x, backend=gpu.name)
    want = np.sum(x, axis=axis, dtype=np.float64).astype(np.float32)
    assert rel_err(t.sum(axis=axis).to_host_buffer(), want) <= 1e-6
    assert np.array_equal(t.max(axis=axis).to_host_buffer(), np.max(x, axis=axis))
    assert np.array_equal(t.argmax(axis).to_host_buffer(), np.argmax(x, axis=axis))


@pytest.mark.parametrize("m,k,n", [(64, 784, 256), (2048, 768, 3072), (128, 9216, 4096), (1000, 17, 3)])
def test_matmul_sizes(gpu, m, k, n):
    r = np.random.default_rng(m + n)
    a = r.standard_normal((m, k)).astype(np.float32)
    b = r.standard_normal((k, n)).astype(np.float32) / np.sqrt(k)
    got = (T.tensor(a, backend=gpu.name) @ T.tensor(b, backend=gpu.name)).to_host_buffer()
    want = (a.astype(np.float64) @ b.astype(np.float64)).astype(np.float32)
    assert_contraction(got, want, lambda: a @ b)


CONV = [((32, 64, 56, 56), (64, 64, 3, 3), 1, 1), ((8, 256, 56, 56), (128, 256, 1, 1), 2, 0),
        ((4, 3, 224, 224), (64, 3, 7, 7), 2, 3), ((8, 3, 224, 224), (64, 3, 11, 11), 4, 2)]


@pytest.mark.parametrize("xs,ws,s,p", CONV)
def test_conv_sizes(gpu, xs, ws, s, p):
    r = np.random.default_rng(xs[1])
    x = r.standard_normal(xs).astype(np.float32)
    w = (r.standard_normal(ws) / np.sqrt(ws[1] * ws[2] * ws[3])).astype(np.float32)
    params = {"stride": (s, s), "padding": (p, p)}
    tx, tw = T.tensor(x, backend=gpu.name), T.tensor(w, backend=gpu.name)
    out = T.conv2d(tx, tw, None, s, p)
    assert_contraction(out.to_host_buffer(), _oracle("conv2d", params, [x, w]),
                       lambda: f32_conv_family(x, w, None, s, p)[0], what="fprop")
    g = r.standard_normal(tuple(out.shape)).astype(np.float32)
    tg = T.tensor(g, backend=gpu.name)
    fam = {}

    def blas(i):
        if "v" not in fam:
            fam["v"] = f32_conv_family(x, w, g, s, p)
        return fam["v"][i]
    gi = T.conv2d_grad_input(tg, tw, xs, s, p).to_host_buffer()
    assert_contraction(gi, _oracle("conv2d_grad_input", dict(params, x_shape=xs), [g, w]), lambda: blas(1),
                       what="dgrad")
    gw = T.conv2d_grad_weight(tx, tg, ws, s, p).to_host_buffer()  # reduces over N*Ho*Wo (up to 100352)
    assert_contraction(gw, _oracle("conv2d_grad_weight", dict(params, w_shape=ws), [x, g]), lambda: blas(2),
                       what="wgrad")


def test_times_one_is_a_broadcast_view(gpu):
    """full(shape, 1) * g (the reference's sum backward spread) is a zero-copy view of g,
    bit-identical to the multiply, and every consumer reads it correctly."""
    r = np.random.default_rng(3)
    g = np.concatenate([r.standard_normal(23), [np.inf, -np.inf, -0.0, 0.0, np.nan]]).astype(np.float32)
    g = g.reshape(2, 1, 14, 1)
    tg = T.tensor(g, backend=gpu.name)
    ones = T.full((2, 3, 14, 5), 1.0, dtype="f32", backend=gpu.name)
    for prod, want in ((ones * tg, np.ones((2, 3, 14, 5), np.float32) * g),
                       (tg * ones, g * np.ones((2, 3, 14, 5), np.float32))):
        assert prod.adapter.block is tg.adapter.block  # no new allocation
        got = prod.to_host_buffer()
        assert np.array_equal(got, want, equal_nan=True)
        assert np.array_equal(np.signbit(got), np.signbit(want))
        assert np.array_equal((prod / 5.0).to_host_buffer(), want / np.float32(5.0), equal_nan=True)
        assert np.array_equal(prod.sum(axis=0).to_host_buffer(),
                              np.sum(want, axis=0, dtype=np.float64).astype(np.float32), equal_nan=True)
    # anything but an exact f32 one keeps the multiply
    twos = T.full((2, 3, 14, 5), 2.0, dtype="f32", backend=gpu.name)
    assert (twos * tg).adapter.block is not tg.adapter.block


def test_fast_division_is_ieee_exact(gpu):
    """The per-row broadcast kernel divides by reciprocal + one exact-residual correction
    (csrc/elementwise.cu div_rn_rcp); it must equal IEEE division bit for bit: 2^26 random
    bit patterns, every mantissa of the divisor against 8 dividends, and the edge exponents."""
    r = np.random.default_rng(11)
    n = 1 << 26
    a = r.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32).view(np.float32)
    b = r.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32).view(np.float32)
    mant = (np.arange(1 << 23, dtype=np.uint32) | np.uint32(127 << 23)).view(np.float32)
    for dividend in (1.0, 1.5, 1.9999999, 3.0, 1.0000001, 1.2345678, 7.654321e-30, 6.5e35):
        a = np.concatenate([a, np.full(mant.size, dividend, np.float32)])
        b = np.concatenate([b, mant])
    edge = np.array([2.0 ** e for e in range(-149, 128)] + [np.inf, -np.inf, np.nan, 0.0, -0.0], np.float32)
    ea, eb = np.meshgrid(edge, edge * np.float32(1.0000001))
    a = np.concatenate([a, ea.ravel(), edge])
    b = np.concatenate([b, eb.ravel(), np.float32(3.0) * edge])
    with np.errstate(all="ignore"):
        want = a / b
    ta, tb = T.tensor(a, backend=gpu.name), T.tensor(b, backend=gpu.name)
    out = T.tensor(np.zeros_like(a), backend=gpu.name)
    gpu._lib.pb_fastdiv_probe(ta.adapter.ptr, tb.adapter.ptr, out.adapter.ptr, a.size)
    got = out.numpy()
    bad = ~((got.view(np.uint32) == want.view(np.uint32)) | (np.isnan(got) & np.isnan(want)))
    assert not bad.any(), (int(bad.sum()), a[bad][:5], b[bad][:5], got[bad][:5], want[bad][:5])


@pytest.mark.parametrize("op", ["add", "sub", "mul", "div"])
@pytest.mark.parametrize("left", [False, True])
def test_row_broadcast_kernel_bit_exact(gpu, op, left):
    """BatchNorm's [N,C,H,W] (op) [1,C,1,1] shapes, either side: the per-row kernel
    (ew_chan4) against numpy's f32 arithmetic, bit for bit."""
    r = np.random.default_rng(5)
    x = r.standard_normal((4, 64, 28, 28)).astype(np.float32)
    m = (r.standard_normal((1, 64, 1, 1)) + 3).astype(np.float32)
    tx, tm = T.tensor(x, backend=gpu.name), T.tensor(m, backend=gpu.name)
    f = {"add": lambda u, v: u + v, "sub": lambda u, v: u - v, "mul": lambda u, v: u * v,
         "div": lambda u, v: u / v}[op]
    got = (f(tm, tx) if left else f(tx, tm)).numpy()
    want = f(m, x) if left else f(x, m)
    assert got.dtype == np.float32 and np.array_equal(got, want)
