"""The drop-in proven on the reference itself: ``GpuBackend`` registered into minml's OWN
registry (paper_2201_12465_b200.gpu.minml_plugin.install, minml/registry.py:149-187), and
minml's own Tensor / Variable / nn / optim / training code -- not this package's front end --
trains on the B200 and matches minml's own EagerBackend on the same inputs and seeds.

minml comes from baseline/_ref (the unmodified reference, installed by
``__graft_entry__.build()`` from /root/reference; it travels to the GPU box with the repo)."""

import collections
import gc
import os
import sys

import numpy as np
import pytest

from golden_util import rel_err

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def minml():
    if not os.path.isdir(os.path.join(REF, "minml")):
        pytest.fail("baseline/_ref/minml missing: run __graft_entry__.build() in the build container")
    sys.path.insert(0, REF)
    import minml
    import minml.autograd  # noqa: F401
    import minml.data  # noqa: F401
    import minml.models  # noqa: F401
    import minml.training  # noqa: F401
    import minml.memory  # noqa: F401
    import minml.wrappers  # noqa: F401
    assert os.path.dirname(minml.__file__).startswith(REF), minml.__file__
    return minml


@pytest.fixture
def pair(minml, request):
    """(gpu, cpu): the B200 backend and minml's EagerBackend, both in minml's registry."""
    from minml.eager import EagerBackend
    from paper_2201_12465_b200.gpu.minml_plugin import install
    tag = request.node.name.replace("[", "-").replace("]", "")
    gpu = install(minml, name=f"b200-{tag}", default=False)
    cpu = EagerBackend(name=f"cpu-{tag}")
    minml.registry.register(cpu)
    yield gpu, cpu
    minml.registry.unregister(gpu.name)
    minml.registry.unregister(cpu.name)


def _train(minml, model_fn, backend, batches, steps, sgd, seed):
    backend.seed(seed)
    model = model_fn(backend.name)
    opt = minml.optim.SGD(model.params(), **sgd)
    losses = [minml.training.train_step(model, *batches[k % len(batches)], opt)[0] for k in range(steps)]
    return losses, [p.numpy() for p in model.params()]


def test_backend_is_a_minml_backend(minml, pair):
    gpu, _ = pair
    assert isinstance(gpu, minml.registry.Backend)
    assert minml.registry.get(gpu.name) is gpu
    t = minml.tensor(np.arange(6, dtype=np.float32).reshape(2, 3), backend=gpu.name)
    assert t.dtype is minml.dtypes.f32  # minml's own DType on minml's own Tensor
    assert np.array_equal((t * 2 + 1).numpy(), np.arange(6, dtype=np.float32).reshape(2, 3) * 2 + 1)


@pytest.mark.parametrize("model", ["mlp", "mnist_cnn"])
def test_minml_training_on_b200_matches_minml_cpu(minml, pair, model):
    """minml.models + minml.optim.SGD + minml.training.train_step, 5 steps on each backend."""
    gpu, cpu = pair
    r = np.random.default_rng(3)
    if model == "mlp":
        fn = lambda be: minml.models.mlp(784, 128, 10, backend=be)  # noqa: E731
        shape = (784,)
    else:
        fn = lambda be: minml.models.mnist_cnn(backend=be)  # noqa: E731
        shape = (1, 28, 28)
    batches = [(r.standard_normal((32,) + shape).astype(np.float32), r.integers(0, 10, 32).astype(np.int64))
               for _ in range(2)]
    sgd = dict(lr=0.05, momentum=0.9)
    lg, pg = _train(minml, fn, gpu, batches, 5, sgd, 7)
    lc, pc = _train(minml, fn, cpu, batches, 5, sgd, 7)
    assert rel_err(lg, lc) <= 1e-5, (lg, lc)
    for a, b in zip(pg, pc):
        assert rel_err(a, b) <= 1e-5


def test_reference_swap_acceptance_on_b200(minml, pair):
    """T/test_acceptance.py:289-335 with the B200 backend inside minml's CountingBackend and a
    RecordingManager ledger: every executed op allocates its output through the attached
    manager tagged with the op, and a second B200 backend with the same seed reproduces the
    logits bit for bit."""
    from paper_2201_12465_b200.gpu.minml_plugin import backend_class
    gpu, _ = pair
    counter = minml.wrappers.CountingBackend(gpu, name=gpu.name + "-counter", seed=5)
    twin = backend_class(minml)(name=gpu.name + "-twin", seed=5)
    minml.registry.register(counter)
    minml.registry.register(twin)
    recorder = minml.memory.RecordingManager(minml.memory.NativeManager())
    counter.attach_manager(recorder)
    try:
        blobs = minml.data.synth_blobs(16, seed=4, shape=(1, 28, 28))
        images = np.stack([blobs[k][0] for k in range(16)])
        labels = np.array([blobs[k][1] for k in range(16)], dtype=np.int64)
        T, V = minml._tensor, minml.autograd.Variable
        model = minml.models.mnist_cnn(backend=counter.name)
        out = model(V(T.tensor(images, backend=counter.name)))
        loss = minml.nn.cross_entropy(out, T.tensor(labels, backend=counter.name))
        loss.backward()
        logits = out.numpy()
        counts = dict(counter.counts)
        tags = collections.Counter(line.split()[3] for line in recorder.lines if line.startswith("A"))
        twin_logits = minml.models.mnist_cnn(backend=twin.name)(V(T.tensor(images, backend=twin.name))).numpy()
        del model, out, loss
        gc.collect()
        gpu.synchronize()
        counter.detach_manager()
    finally:
        minml.registry.unregister(counter.name)
        minml.registry.unregister(twin.name)
    for op in ("add", "maximum", "matmul", "conv2d"):
        assert counts.get(op, 0) > 0 and counts[op] == tags[op], (op, counts.get(op), tags[op])
    assert np.array_equal(logits, twin_logits)


def test_minml_errors_cross_the_boundary(minml, pair):
    gpu, _ = pair
    a = minml.tensor(np.array([1, 2, 3], np.int32), backend=gpu.name)
    b = minml.tensor(np.array([1, 0, 3], np.int32), backend=gpu.name)
    with pytest.raises(minml.errors.DomainError):
        (a / b).numpy()
    with pytest.raises(minml.errors.DomainError):
        (a / 0).numpy()


def test_minml_memory_manager_ledger_is_exact(minml, pair):
    """minml's own CachingManager attached to the B200 backend keeps an exact ledger."""
    gpu, _ = pair
    mgr = minml.memory.make_manager("caching")
    gpu.attach_manager(mgr)
    model = minml.models.mlp(16, 12, 10, backend=gpu.name)
    opt = minml.optim.SGD(model.params(), lr=0.1)
    r = np.random.default_rng(0)
    for _ in range(3):
        minml.training.train_step(model, r.standard_normal((10, 16)).astype(np.float32),
                                  r.integers(0, 10, 10).astype(np.int64), opt)
    del model, opt
    gc.collect()
    gpu.synchronize()
    s = mgr.stats()
    assert s.live_bytes_requested == 0 and s.alloc_count > 0
    gpu.detach_manager()


@pytest.mark.parametrize("name", ["lenet_full", "resnet50_full"])
def test_minml_front_end_fullsize_on_b200(minml, pair, name):
    """minml's own front end driving full-size configs on the B200 reproduces minml's CPU
    trajectory (tests/golden/fullsize.*): the same bar as the product front end."""
    from fullsize_util import BUILDERS, arrays, batches, check, compare, meta
    from paper_2201_12465_b200 import models as PM
    gpu, _ = pair
    ns = PM.namespace(minml.nn, minml.ops, minml._tensor, minml.autograd)
    m = meta()[name]
    fns = {"lenet_full": lambda be: PM.mnist_cnn(backend=be, ns=ns),
           "resnet50_full": lambda be: PM.resnet50(backend=be, ns=ns)}
    assert name in BUILDERS
    losses, params = _train(minml, fns[name], gpu, batches(name, m["batch"]), m["steps"], m["sgd"], m["seed"])
    err = compare(name, m, arrays(), losses, params)
    check(err, m)
