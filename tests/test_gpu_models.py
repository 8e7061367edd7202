"""End-to-end parity on the B200: the five config families' reduced trajectories through
the product front end + CUDA backend vs the reference's own run (tests/golden/models.json),
the backend-swap check of T/test_acceptance.py:289-335, and allocator conservation."""

import gc
import json
import os

import numpy as np
import pytest

from frontend_util import BUILDERS, run_trajectory
from golden_util import models_meta, rel_err
from gpu_util import gpu_backend
from paper_2201_12465_b200 import _tensor as T
from paper_2201_12465_b200 import memory, models, nn, registry
from paper_2201_12465_b200.autograd import Variable
from paper_2201_12465_b200.gpu.backend import GpuBackend
from paper_2201_12465_b200.wrappers import CountingBackend

pytestmark = pytest.mark.gpu
META = models_meta()
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "models_sensitivity.json")) as _f:
    SENS = json.load(_f)  # tests/golden/make_models_sensitivity.py


@pytest.mark.parametrize("name", sorted(BUILDERS))
def test_trajectory_matches_reference(name):
    be = gpu_backend()
    meta = META[name]
    losses, sums, _ = run_trajectory(name, meta, be)
    # north-star tolerance (BASELINE.json): loss trajectories within 1e-3
    sens = SENS[name]  # the reference's own gaps under a 1e-7 init perturbation
    assert rel_err(losses, meta["losses"]) <= max(1e-3, 2 * sens["loss"]), (losses, meta["losses"])
    # every parameter's signed sum and sum|p| under the reference's metric (the batch-4
    # BatchNorm ResNet's cancelling signed sums move 1.9e-2 in the reference itself)
    assert rel_err(sums, meta["param_sums"]) <= max(1e-3, 2 * sens["sums"]), (name, sums, meta["param_sums"])


@pytest.mark.parametrize("name", sorted(BUILDERS))
def test_trajectory_f64_accumulation_path_is_tight(name):
    """With the SIMT contractions (f32 products accumulated in f64, like the reference)
    every parameter sum matches the reference run to 1e-3 with the reference's metric."""
    be = gpu_backend()
    meta = META[name]
    be._lib.pb_set_gemm_path(0)
    try:
        losses, sums, _ = run_trajectory(name, meta, be)
    finally:
        be._lib.pb_set_gemm_path(2)
    assert rel_err(losses, meta["losses"]) <= 1e-3, (losses, meta["losses"])
    assert rel_err(sums, meta["param_sums"]) <= 1e-3


def test_fused_sgd_updates_in_place_after_first_step():
    be = gpu_backend()
    meta = META["mlp"]
    run_trajectory("mlp", dict(meta, steps=3), be)
    assert be.last_sgd["rebound"] == 0, be.last_sgd


def test_counting_wrapper_sees_every_op_and_swap_is_bit_exact():
    inner = GpuBackend(name="gpu-count-inner")
    counter = CountingBackend(inner, name="gpu-counter", seed=5)
    twin = GpuBackend(name="gpu-twin", seed=5)
    registry.register(counter)
    registry.register(twin)
    try:
        rng = np.random.default_rng(4)
        images = rng.standard_normal((16, 1, 28, 28)).astype(np.float32)
        labels = rng.integers(0, 10, 16).astype(np.int64)
        model = models.mnist_cnn(backend=counter.name)
        out = model(Variable(T.tensor(images, backend=counter.name)))
        loss = nn.cross_entropy(out, T.tensor(labels, backend=counter.name))
        loss.backward()
        logits = out.numpy()
        twin_out = models.mnist_cnn(backend=twin.name)(Variable(T.tensor(images, backend=twin.name)))
        assert np.array_equal(logits, twin_out.numpy())
        for op in ("add", "maximum", "matmul", "conv2d", "conv2d_grad_weight"):
            assert counter.counts[op] > 0
    finally:
        registry.unregister(counter.name)
        registry.unregister(twin.name)


def test_allocator_conservation_on_device():
    be = GpuBackend(name="gpu-conserve", seed=3)
    registry.register(be)
    mgr = memory.make_manager("caching")
    be.attach_manager(mgr)
    try:
        model = models.mlp(16, 12, 10, backend=be.name)
        from paper_2201_12465_b200 import optim, training
        opt = optim.SGD(model.params(), lr=0.1)
        r = np.random.default_rng(0)
        for _ in range(3):
            training.train_step(model, r.standard_normal((10, 16)).astype(np.float32),
                                r.integers(0, 10, 10).astype(np.int64), opt)
        del model, opt
        gc.collect()
        be.synchronize()
        mgr.flush_cache()
        s = mgr.stats()
        assert s.live_bytes_requested == 0 and s.cache_bytes == 0 and s.alloc_count == s.free_count > 0
        be.detach_manager()
    finally:
        registry.unregister(be.name)
