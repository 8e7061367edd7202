"""Model builders for the five BASELINE.json configs.

``mlp`` and ``mnist_cnn`` restate minml/models.py:6-34.  AlexNet, ResNet-50
and the BERT-base-like encoder have no builder in the reference; they are
composed here from reference-API modules exactly as SURVEY §8(d2) lists.

Every builder takes ``ns`` — the namespace whose ``nn``/``ops``/``T``/
``autograd`` modules it composes.  The default is this package; the golden
fixture generator (tests/golden/make_golden.py) passes the reference's own
``minml`` modules, so both sides run the identical composition.
"""

import math
import types


def _default_ns():
    from . import _tensor, autograd, nn, ops
    return types.SimpleNamespace(nn=nn, ops=ops, T=_tensor, autograd=autograd)


def namespace(nn, ops, T, autograd):
    return types.SimpleNamespace(nn=nn, ops=ops, T=T, autograd=autograd)


_LIBS = {}


def library(ns=None):
    """Composite modules built over one namespace (cached per namespace)."""
    ns = ns or _default_ns()
    key = id(ns.nn)
    lib = _LIBS.get(key)
    if lib is None:
        lib = _LIBS[key] = _build_library(ns)
    return lib


def _build_library(ns):
    nn, ops, T, ag = ns.nn, ns.ops, ns.T, ns.autograd
    Variable = ag.Variable

    class PadMaxPool(nn.Module):
        """ResNet stem pool: pad H,W with -inf, then MaxPool2D(k, s)."""

        def __init__(self, kernel=3, stride=2, pad=1):
            super().__init__()
            self.pool = self.register_child("pool", nn.MaxPool2D(kernel, stride))
            self.pad = pad

        def forward(self, x):
            p = self.pad
            return self.pool(x.pad(((0, 0), (0, 0), (p, p), (p, p)), value=-math.inf))

    class Bottleneck(nn.Module):
        expansion = 4

        def __init__(self, cin, width, stride, backend, dtype):
            super().__init__()
            cout = width * 4
            mk = dict(bias=False, dtype=dtype, backend=backend)
            self.c1 = self.register_child("c1", nn.Conv2D(cin, width, 1, **mk))
            self.b1 = self.register_child("b1", nn.BatchNorm(width, dtype=dtype, backend=backend))
            self.c2 = self.register_child("c2", nn.Conv2D(width, width, 3, stride, 1, **mk))
            self.b2 = self.register_child("b2", nn.BatchNorm(width, dtype=dtype, backend=backend))
            self.c3 = self.register_child("c3", nn.Conv2D(width, cout, 1, **mk))
            self.b3 = self.register_child("b3", nn.BatchNorm(cout, dtype=dtype, backend=backend))
            self.proj = None
            if stride != 1 or cin != cout:
                self.proj = self.register_child("proj", nn.Conv2D(cin, cout, 1, stride, **mk))
                self.bp = self.register_child("bp", nn.BatchNorm(cout, dtype=dtype, backend=backend))

        def forward(self, x):
            h = ops.relu(self.b1(self.c1(x)))
            h = ops.relu(self.b2(self.c2(h)))
            h = self.b3(self.c3(h))
            sc = x if self.proj is None else self.bp(self.proj(x))
            return ops.relu(h + sc)

    class GlobalAvgPool(nn.Module):
        def forward(self, x):
            return x.mean(axis=3).mean(axis=2)

    class LayerNorm(nn.Module):
        """Normalise the last axis: (x - mean)/sqrt(var + eps) * gamma + beta."""

        def __init__(self, d, eps=1e-5, dtype="f32", backend=None):
            super().__init__()
            self.eps = eps
            self.gamma = self.register_param("gamma", Variable(T.ones((d,), dtype=dtype, backend=backend), requires_grad=True))
            self.beta = self.register_param("beta", Variable(T.zeros((d,), dtype=dtype, backend=backend), requires_grad=True))

        def forward(self, x):
            mu = x.mean(axis=-1, keepdims=True)
            c = x - mu
            var = (c * c).mean(axis=-1, keepdims=True)
            return c / (var + self.eps).sqrt() * self.gamma + self.beta

    class EncoderLayer(nn.Module):
        def __init__(self, d, heads, ffn, seq, backend, dtype):
            super().__init__()
            self.d, self.h, self.s = d, heads, seq
            mk = dict(dtype=dtype, backend=backend)
            self.q = self.register_child("q", nn.Linear(d, d, **mk))
            self.k = self.register_child("k", nn.Linear(d, d, **mk))
            self.v = self.register_child("v", nn.Linear(d, d, **mk))
            self.o = self.register_child("o", nn.Linear(d, d, **mk))
            self.ln1 = self.register_child("ln1", LayerNorm(d, **mk))
            self.f1 = self.register_child("f1", nn.Linear(d, ffn, **mk))
            self.f2 = self.register_child("f2", nn.Linear(ffn, d, **mk))
            self.ln2 = self.register_child("ln2", LayerNorm(d, **mk))

        def _heads(self, t, b):
            return t.reshape((b, self.s, self.h, self.d // self.h)).transpose((0, 2, 1, 3)).reshape(
                (b * self.h, self.s, self.d // self.h))

        def forward(self, x):
            b = x.shape[0] // self.s
            dh = self.d // self.h
            q, k, v = self._heads(self.q(x), b), self._heads(self.k(x), b), self._heads(self.v(x), b)
            scores = ag.matmul(q, k.transpose((0, 2, 1))) * (1.0 / math.sqrt(dh))
            ctx = ag.matmul(ops.softmax(scores, axis=-1), v)
            ctx = ctx.reshape((b, self.h, self.s, dh)).transpose((0, 2, 1, 3)).reshape((b * self.s, self.d))
            x = self.ln1(x + self.o(ctx))
            return self.ln2(x + self.f2(ops.gelu(self.f1(x))))

    class BertLike(nn.Module):
        """one_hot(tokens) @ E + P -> LN -> encoder layers -> CLS Linear -> LogSoftmax."""

        def __init__(self, vocab, seq, d, heads, ffn, layers, classes, backend, dtype):
            super().__init__()
            self.vocab, self.seq, self.d = vocab, seq, d
            self.emb = self.register_param("emb", Variable(
                nn.uniform_init((vocab, d), d, dtype, backend) if hasattr(nn, "uniform_init")
                else nn._uniform_init((vocab, d), d, dtype, backend), requires_grad=True))
            self.pos = self.register_param("pos", Variable(
                nn.uniform_init((seq, d), d, dtype, backend) if hasattr(nn, "uniform_init")
                else nn._uniform_init((seq, d), d, dtype, backend), requires_grad=True))
            self.ln = self.register_child("ln", LayerNorm(d, dtype=dtype, backend=backend))
            self.layers = [self.register_child(f"l{i}", EncoderLayer(d, heads, ffn, seq, backend, dtype))
                           for i in range(layers)]
            self.head = self.register_child("head", nn.Linear(d, classes, dtype=dtype, backend=backend))
            self.dtype = dtype

        def forward(self, tokens):
            t = tokens.data if isinstance(tokens, Variable) else tokens
            b = t.shape[0]
            flat = t.reshape((b * self.seq,))
            oh = Variable(ops.one_hot(flat, self.vocab, dtype=self.dtype))
            x = ag.matmul(oh, self.emb).reshape((b, self.seq, self.d)) + self.pos
            x = self.ln(x.reshape((b * self.seq, self.d)))
            for layer in self.layers:
                x = layer(x)
            cls = x.reshape((b, self.seq, self.d)).slice((0, 0, 0), (b, 1, self.d)).reshape((b, self.d))
            return ops.log_softmax(self.head(cls), -1)

    return types.SimpleNamespace(PadMaxPool=PadMaxPool, Bottleneck=Bottleneck, GlobalAvgPool=GlobalAvgPool,
                                 LayerNorm=LayerNorm, EncoderLayer=EncoderLayer, BertLike=BertLike)


def mlp(in_dim, hidden, classes, backend=None, dtype="f32", ns=None):
    nn = (ns or _default_ns()).nn
    return nn.Sequential(nn.Linear(in_dim, hidden, dtype=dtype, backend=backend), nn.ReLU(),
                         nn.Linear(hidden, classes, dtype=dtype, backend=backend), nn.LogSoftmax())


def mnist_cnn(backend=None, dtype="f32", ns=None):
    nn = (ns or _default_ns()).nn
    mk = dict(dtype=dtype, backend=backend)
    return nn.Sequential(
        nn.Conv2D(1, 32, 5, **mk), nn.ReLU(), nn.MaxPool2D(2),
        nn.Conv2D(32, 64, 5, **mk), nn.ReLU(), nn.MaxPool2D(2),
        nn.View((1024,)),
        nn.Linear(1024, 128, **mk), nn.ReLU(), nn.Linear(128, 10, **mk), nn.LogSoftmax())


def alexnet(classes=1000, image=224, channels=(64, 192, 384, 256, 256), hidden=4096, dropout=0.5,
            backend=None, dtype="f32", ns=None):
    nn = (ns or _default_ns()).nn
    mk = dict(dtype=dtype, backend=backend)
    c1, c2, c3, c4, c5 = channels
    s = (image + 4 - 11) // 4 + 1
    s = (s - 3) // 2 + 1
    s = (s - 3) // 2 + 1
    s = (s - 3) // 2 + 1
    flat = c5 * s * s
    return nn.Sequential(
        nn.Conv2D(3, c1, 11, 4, 2, **mk), nn.ReLU(), nn.MaxPool2D(3, 2),
        nn.Conv2D(c1, c2, 5, 1, 2, **mk), nn.ReLU(), nn.MaxPool2D(3, 2),
        nn.Conv2D(c2, c3, 3, 1, 1, **mk), nn.ReLU(),
        nn.Conv2D(c3, c4, 3, 1, 1, **mk), nn.ReLU(),
        nn.Conv2D(c4, c5, 3, 1, 1, **mk), nn.ReLU(), nn.MaxPool2D(3, 2),
        nn.View((flat,)), nn.Dropout(dropout),
        nn.Linear(flat, hidden, **mk), nn.ReLU(), nn.Dropout(dropout),
        nn.Linear(hidden, hidden, **mk), nn.ReLU(),
        nn.Linear(hidden, classes, **mk), nn.LogSoftmax())


def resnet50(classes=1000, layers=(3, 4, 6, 3), width=64, backend=None, dtype="f32", ns=None):
    """ResNet-50 v1.5 (stride on the 3x3), no conv bias, composed BatchNorm; 25.56M params."""
    ns = ns or _default_ns()
    nn, lib = ns.nn, library(ns)
    mk = dict(dtype=dtype, backend=backend)
    mods = [nn.Conv2D(3, width, 7, 2, 3, bias=False, **mk), nn.BatchNorm(width, **mk), nn.ReLU(),
            lib.PadMaxPool(3, 2, 1)]
    cin = width
    for stage, n in enumerate(layers):
        w = width * (2 ** stage)
        for i in range(n):
            mods.append(lib.Bottleneck(cin, w, 2 if (i == 0 and stage > 0) else 1, backend, dtype))
            cin = w * 4
    mods += [lib.GlobalAvgPool(), nn.Linear(cin, classes, **mk), nn.LogSoftmax()]
    return nn.Sequential(*mods)


def bert_base(vocab=30522, seq=128, d=768, heads=12, ffn=3072, layers=12, classes=2,
              backend=None, dtype="f32", ns=None):
    """BERT-base-like encoder classifier, 108.6M params at the defaults."""
    ns = ns or _default_ns()
    return library(ns).BertLike(vocab, seq, d, heads, ffn, layers, classes, backend, dtype)


CONFIGS = {
    "mlp": dict(build=lambda be: mlp(784, 256, 10, backend=be), input=(784,), classes=10, batch=64,
                sgd=dict(lr=0.05)),
    "lenet": dict(build=lambda be: mnist_cnn(backend=be), input=(1, 28, 28), classes=10, batch=128,
                  sgd=dict(lr=0.05)),
    "alexnet": dict(build=lambda be: alexnet(backend=be), input=(3, 224, 224), classes=1000, batch=128,
                    sgd=dict(lr=0.01, momentum=0.9)),
    "resnet50": dict(build=lambda be: resnet50(backend=be), input=(3, 224, 224), classes=1000, batch=32,
                     sgd=dict(lr=0.1, momentum=0.9)),
    "bert": dict(build=lambda be: bert_base(backend=be), input=None, tokens=(128, 30522), classes=2,
                 batch=16, sgd=dict(lr=0.01, momentum=0.9)),
}
