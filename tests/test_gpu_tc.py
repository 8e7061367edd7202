"""Parity of the tcgen05 3xTF32 contraction kernels (csrc/gemm_tc.cu) against the f64
reference contraction (minml/kernels.py:166-239 computes f32 matmul/conv in f64 and
rounds once), on every code path the dispatcher can take: row-/k-mode operand loaders,
vectorised and scalar gathers, strided convs, stride-2 dgrad, split-K wgrad and matmul,
batched matmul, transposed views, ragged tiles.

Tolerance: the reference's metric |a-b|/max(|a|,|b|,1) <= 1e-5 (T/test_acceptance.py:260-262),
through golden_util.assert_contraction: where a long K-reduction of O(1) terms cancels below
what any f32-accumulating GEMM resolves, the kernel must instead beat numpy's own f32 BLAS on
the same operands by 2x under that metric (see its docstring)."""

import numpy as np
import pytest

from golden_util import assert_contraction, contraction_err, f32_conv_family
from gpu_util import gpu_backend
from paper_2201_12465_b200 import _tensor as T

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.fixture(scope="module")
def gpu():
    be = gpu_backend()
    assert be._lib.pb_gemm_path() == 2
    return be


@pytest.fixture(params=[2, 1], ids=["tma", "simt-fed"])
def path(request, gpu):
    """Both tcgen05 kernel families: TMA-fed (gemm_tma.cu) and SIMT-fed (gemm_tc.cu)."""
    gpu._lib.pb_set_gemm_path(request.param)
    yield request.param
    gpu._lib.pb_set_gemm_path(2)


def _np_conv(x, w, s, p):
    """f64 direct convolution (cross-correlation), NCHW."""
    n, c, h, wd = x.shape
    f, _, kh, kw = w.shape
    xp = np.pad(x.astype(np.float64), ((0, 0), (0, 0), (p, p), (p, p)))
    ho, wo = (h + 2 * p - kh) // s + 1, (wd + 2 * p - kw) // s + 1
    cols = np.empty((n, c, kh, kw, ho, wo))
    for r in range(kh):
        for t in range(kw):
            cols[:, :, r, t] = xp[:, :, r:r + s * ho:s, t:t + s * wo:s]
    return np.einsum("ncrshw,fcrs->nfhw", cols, w.astype(np.float64)), cols


def _np_dgrad(g, w, xs, s, p):
    n, c, h, wd = xs
    f, _, kh, kw = w.shape
    ho, wo = g.shape[2], g.shape[3]
    dxp = np.zeros((n, c, h + 2 * p + s, wd + 2 * p + s))
    for r in range(kh):
        for t in range(kw):
            dxp[:, :, r:r + s * ho:s, t:t + s * wo:s] += np.einsum("nfhw,fc->nchw", g.astype(np.float64),
                                                                 w[:, :, r, t].astype(np.float64))
    return dxp[:, :, p:p + h, p:p + wd]


CONVS = [
    # (x shape, w shape, stride, pad)
    ((2, 64, 14, 14), (64, 64, 3, 3), 1, 1),      # C4 fast gather, BN=64
    ((2, 32, 9, 11), (128, 32, 3, 3), 1, 1),      # ragged pixels, BN=128
    ((3, 3, 23, 23), (16, 3, 7, 7), 2, 3),        # stem-like: C=3 scalar gather, K=147
    ((2, 1, 28, 28), (32, 1, 5, 5), 1, 0),        # LeNet conv1: C=1
    ((2, 64, 15, 15), (96, 64, 1, 1), 2, 0),      # 1x1 stride-2 downsample (dgrad stride grid)
    ((1, 128, 8, 8), (200, 128, 3, 3), 2, 1),     # stride-2 3x3, F not a tile multiple
    ((4, 256, 7, 7), (64, 256, 1, 1), 1, 0),      # P = 49 (wgrad scalar g gather)
    ((3, 64, 20, 20), (64, 64, 3, 3), 1, 1),      # im2col walks across rows and images
    ((2, 96, 17, 13), (64, 96, 3, 3), 2, 1),      # odd sizes, stride 2, C = 3 x 32
    ((5, 32, 6, 6), (256, 32, 1, 1), 1, 0),       # 1x1, K tail, F = 2 x BN
    ((2, 160, 9, 9), (96, 160, 3, 3), 1, 2),      # pad 2 (dgrad pad 0), C not a BM multiple
]


@pytest.mark.parametrize("xs,ws,s,p", CONVS, ids=[f"{a}-{b}-s{c}p{d}" for a, b, c, d in CONVS])
def test_conv_family_tc(gpu, path, xs, ws, s, p):
    r = np.random.default_rng(sum(xs) + sum(ws))
    x = r.standard_normal(xs).astype(np.float32)
    w = (r.standard_normal(ws) / np.sqrt(ws[1] * ws[2] * ws[3])).astype(np.float32)
    b = r.standard_normal(ws[0]).astype(np.float32)
    tx, tw, tb = (T.tensor(a, backend=gpu.name) for a in (x, w, b))
    want, cols = _np_conv(x, w, s, p)
    got = T.conv2d(tx, tw, tb, s, p).to_host_buffer()
    y32 = lambda: f32_conv_family(x, w, None, s, p)[0]  # noqa: E731
    assert_contraction(got, (want + b[None, :, None, None]).astype(np.float32),
                       lambda: y32() + b[None, :, None, None], what="fprop+bias")
    got_nb = T.conv2d(tx, tw, None, s, p).to_host_buffer()
    assert_contraction(got_nb, want.astype(np.float32), y32, what="fprop")
    g = r.standard_normal(got.shape).astype(np.float32)
    tg = T.tensor(g, backend=gpu.name)
    gi = T.conv2d_grad_input(tg, tw, xs, s, p).to_host_buffer()
    assert_contraction(gi, _np_dgrad(g, w, xs, s, p).astype(np.float32),
                       lambda: f32_conv_family(x, w, g, s, p)[1], what="dgrad")
    gw = T.conv2d_grad_weight(tx, tg, ws, s, p).to_host_buffer()
    want_w = np.einsum("ncrshw,nfhw->fcrs", cols, g.astype(np.float64))
    assert_contraction(gw, want_w.astype(np.float32), lambda: f32_conv_family(x, w, g, s, p)[2], what="wgrad")


MATMULS = [(64, 784, 256), (64, 256, 10), (256, 64, 10), (784, 64, 256), (1000, 17, 3), (1, 1, 1),
           (130, 4100, 70), (2048, 768, 768)]


@pytest.mark.parametrize("m,k,n", MATMULS)
def test_matmul_layouts_tc(gpu, m, k, n):
    r = np.random.default_rng(m * 7 + k * 3 + n)
    a = r.standard_normal((m, k)).astype(np.float32)
    b = (r.standard_normal((k, n)) / np.sqrt(k)).astype(np.float32)
    want = (a.astype(np.float64) @ b.astype(np.float64)).astype(np.float32)
    ta, tb = T.tensor(a, backend=gpu.name), T.tensor(b, backend=gpu.name)
    blas = lambda: a @ b  # noqa: E731
    assert_contraction((ta @ tb).to_host_buffer(), want, blas)
    # transposed views for both operands (Linear's W^T and matmul backward): no copies
    at = T.tensor(np.ascontiguousarray(a.T), backend=gpu.name).transpose()
    bt = T.tensor(np.ascontiguousarray(b.T), backend=gpu.name).transpose()
    assert_contraction((at @ tb).to_host_buffer(), want, blas)
    assert_contraction((ta @ bt).to_host_buffer(), want, blas)
    assert_contraction((at @ bt).to_host_buffer(), want, blas)


def test_batched_matmul_tc(gpu):
    r = np.random.default_rng(9)
    a = r.standard_normal((6, 128, 64)).astype(np.float32)
    b = r.standard_normal((6, 64, 100)).astype(np.float32) / 8
    want = np.einsum("bmk,bkn->bmn", a.astype(np.float64), b.astype(np.float64)).astype(np.float32)
    ta, tb = T.tensor(a, backend=gpu.name), T.tensor(b, backend=gpu.name)
    assert_contraction((ta @ tb).to_host_buffer(), want, lambda: np.matmul(a, b))
    # attention-style transposed operand: b^T stored as [6,100,64]
    bt = T.tensor(np.ascontiguousarray(np.transpose(b, (0, 2, 1))), backend=gpu.name).transpose((0, 2, 1))
    assert_contraction((ta @ bt).to_host_buffer(), want, lambda: np.matmul(a, b))


def test_tc_matches_simt_path(gpu):
    """The SIMT kernels (f64 accumulation) are the in-library reference for the tc path: the
    tcgen05 families agree with them to 1e-5 of the output scale (all-ones gradients make the
    wgrad sums cancel-free, so this is the plain relative agreement of the two families)."""
    r = np.random.default_rng(4)
    x = r.standard_normal((4, 64, 28, 28)).astype(np.float32)
    w = (r.standard_normal((128, 64, 3, 3)) / 24).astype(np.float32)
    tx, tw = T.tensor(x, backend=gpu.name), T.tensor(w, backend=gpu.name)
    lib = gpu._lib
    outs = []
    for path in (2, 1, 0):
        lib.pb_set_gemm_path(path)
        try:
            for s in (1, 2):
                y = T.conv2d(tx, tw, None, s, 1)
                g = T.tensor(np.ones(y.shape, np.float32), backend=gpu.name)
                outs.append([y.to_host_buffer(), T.conv2d_grad_input(g, tw, x.shape, s, 1).to_host_buffer(),
                             T.conv2d_grad_weight(tx, g, w.shape, s, 1).to_host_buffer()])
        finally:
            lib.pb_set_gemm_path(2)
    n = len(outs) // 3
    for other in (outs[n:2 * n], outs[2 * n:]):
        for a, b in zip(outs[:n], other):
            for u, v in zip(a, b):
                assert contraction_err(u, v) <= TOL


@pytest.mark.parametrize("m,k,n", [(256, 96, 80), (300, 770, 130), (2048, 768, 64), (256, 2048, 96), (512, 67, 257)])
def test_tma_matmul_matches_f64_reference(gpu, m, k, n):
    """pb_matmul_tma (rank 2, M >= 256: operands pre-split into K-major planes from any
    strided view, split-K folded in f64) against the reference's f64 product
    (minml/kernels.py:166-173), for the three operand layouts the autograd issues: x @ W^T,
    g @ W and g^T @ x.  Shapes cover ragged K (padded pitch, zero tails), ragged M/N tiles and
    the split-K path (few tiles, long K)."""
    r = np.random.default_rng(m + k + n)
    a = r.standard_normal((m, k)).astype(np.float32)
    w = (r.standard_normal((n, k)) / np.sqrt(k)).astype(np.float32)
    ta = T.tensor(a, backend=gpu.name)
    tw = T.tensor(w, backend=gpu.name)
    launches0 = gpu.launch_count()
    got = T.matmul(ta, tw.transpose()).to_host_buffer()              # W^T as a strided view
    assert gpu.launch_count() - launches0 >= 3                         # 2 pre-passes + the GEMM
    want = (a.astype(np.float64) @ w.astype(np.float64).T).astype(np.float32)
    assert_contraction(got, want, lambda: a @ w.T, what="x @ W^T")
    g = r.standard_normal((m, n)).astype(np.float32)
    tg = T.tensor(g, backend=gpu.name)
    got = T.matmul(tg, tw).to_host_buffer()                            # [m,n] x [n,k]
    assert_contraction(got, (g.astype(np.float64) @ w.astype(np.float64)).astype(np.float32), lambda: g @ w,
                       what="g @ W")
    if k >= 256:
        got = T.matmul(tg.transpose(), ta).to_host_buffer()           # [n,m] x [m,k], M = n
        want = (g.astype(np.float64).T @ a.astype(np.float64)).astype(np.float32)
        assert_contraction(got, want, lambda: g.T @ a, what="g^T @ x")


@pytest.mark.parametrize("n,c,h,f,s", [(8, 64, 14, 128, 1), (4, 96, 20, 64, 2), (8, 128, 14, 256, 1), (2, 256, 28, 64, 2),
                                       (16, 256, 7, 64, 1)])
def test_wgrad_1x1_gemm_matches_f64_reference(gpu, n, c, h, f, s):
    """pb_conv2d_grad_weight_mm: 1x1 grad_weight (minml/kernels.py:231-239) as a TMA GEMM over
    K = N*HO*WO, with the larger channel count on the TMEM lanes, stride 1 and 2, against
    the f64 sum over the gradient grid."""
    r = np.random.default_rng(n * c + h + f + s)
    x = r.standard_normal((n, c, h, h)).astype(np.float32)
    ho = (h - 1) // s + 1
    g = r.standard_normal((n, f, ho, ho)).astype(np.float32)
    tx, tg = T.tensor(x, backend=gpu.name), T.tensor(g, backend=gpu.name)
    got = T.conv2d_grad_weight(tx, tg, (f, c, 1, 1), s, 0).to_host_buffer()
    xs = x[:, :, ::s, ::s].astype(np.float64)
    want = np.einsum("nfhw,nchw->fc", g.astype(np.float64), xs).astype(np.float32)[:, :, None, None]
    blas = lambda: np.tensordot(g, xs.astype(np.float32), axes=([0, 2, 3], [0, 2, 3]))[:, :, None, None]  # noqa: E731
    assert_contraction(got, want, blas, what="1x1 wgrad")


def _np_dgrad(g, w, xshape, s, p):
    """f64 adjoint of the strided cross-correlation: scatter every tap's contribution."""
    n, c, h, wd = xshape
    _, _, kh, kw = w.shape
    ho, wo = g.shape[2], g.shape[3]
    dx = np.zeros((n, c, h + 2 * p + s, wd + 2 * p + s))
    g64, w64 = g.astype(np.float64), w.astype(np.float64)
    for r in range(kh):
        for q in range(kw):
            dx[:, :, r:r + s * ho:s, q:q + s * wo:s] += np.einsum("nfhw,fc->nchw", g64, w64[:, :, r, q])
    return dx[:, :, p:p + h, p:p + wd].astype(np.float32)


@pytest.mark.parametrize("n,c,h,f,k,s,p", [(4, 64, 16, 64, 3, 2, 1), (2, 128, 15, 96, 3, 2, 1), (2, 32, 14, 64, 5, 2, 2),
                                           (2, 64, 13, 32, 3, 3, 1), (3, 96, 12, 128, 4, 2, 1)])
def test_subpixel_dgrad_matches_f64_reference(gpu, n, c, h, f, k, s, p):
    """Strided k x k grad_input by sub-pixel decomposition (one stride-1 TMA implicit GEMM per
    output phase class, asymmetric halos, scattered into dx; minml/kernels.py:213-228)
    against the f64 adjoint, including odd extents, k = 4 and 5, and stride 3."""
    r = np.random.default_rng(n + c + h + f + k + s)
    ho = (h + 2 * p - k) // s + 1
    g = r.standard_normal((n, f, ho, ho)).astype(np.float32)
    w = (r.standard_normal((f, c, k, k)) / np.sqrt(f * k * k)).astype(np.float32)
    got = T.conv2d_grad_input(T.tensor(g, backend=gpu.name), T.tensor(w, backend=gpu.name), (n, c, h, h), s,
                              p).to_host_buffer()
    assert_contraction(got, _np_dgrad(g, w, (n, c, h, h), s, p),
                       lambda: f32_conv_family(np.zeros((n, c, h, h), np.float32), w, g, s, p)[1], what="dgrad")
