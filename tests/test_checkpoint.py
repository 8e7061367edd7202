"""Checkpoint and module-stream I/O (minml/nn.py:444-590,
minml/training.py:119-214) against a file the reference itself wrote
(tests/golden/checkpoint.mnck, made by make_checkpoint_golden.py): this framework must read
it bit-exactly and write the identical bytes back, on the CPU oracle backend and, through
to_host/from_host, on the B200 backend."""

import os

import numpy as np
import pytest

from gpu_util import gpu_backend
from oracle.backend import OracleBackend
from paper_2201_12465_b200 import errors, nn, optim, registry, training

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "checkpoint.mnck")


@pytest.fixture
def oracle(request):
    be = OracleBackend(name=f"ckpt-{request.node.name}")
    registry.register(be)
    yield be
    registry.unregister(be.name)


def _gold():
    with open(GOLD, "rb") as f:
        return f.read()


def _resave(be, tmp_path):
    ck = training.load_checkpoint(GOLD, backend=be.name)
    opt = ck.restore_optimizer()
    ck.restore_rng(be.name)
    out = tmp_path / "again.mnck"
    training.save_checkpoint(out, ck.model, opt, epoch=ck.epoch, extra=ck.extra)
    return ck, opt, out.read_bytes()


def test_reference_checkpoint_round_trips_byte_identical(oracle, tmp_path):
    ck, opt, again = _resave(oracle, tmp_path)
    assert ck.epoch == 2 and ck.extra == {"note": "golden"}
    assert [type(m).kind for _, m in ck.model._children] == [
        "conv2d", "batch_norm", "relu", "max_pool2d", "view", "dropout", "linear", "log_softmax"]
    assert opt.momentum == 0.9 and len(opt.state_entries()) == len(opt.params)
    assert again == _gold()


def test_module_stream_round_trip_and_corruption(oracle, tmp_path):
    ck = training.load_checkpoint(GOLD, backend=oracle.name)
    blob = nn.serialize(ck.model)
    clone = nn.deserialize(blob, backend=oracle.name)
    for a, b in zip(ck.model.params(), clone.params()):
        assert np.array_equal(a.numpy(), b.numpy())
    assert nn.serialize(clone) == blob
    path = tmp_path / "m.mnnb"
    nn.save_module(clone, path)
    assert nn.serialize(nn.load_module(path, backend=oracle.name)) == blob
    for bad in (b"XXXX" + blob[4:], blob[:-3], blob + b"\x00"):
        with pytest.raises(errors.FormatError):
            nn.deserialize(bad, backend=oracle.name)
    gold = _gold()
    for bad in (b"XXXX" + gold[4:], gold[:-1], gold + b"\x00"):
        p = tmp_path / "bad.mnck"
        p.write_bytes(bad)
        with pytest.raises(errors.FormatError):
            training.load_checkpoint(p, backend=oracle.name)


def test_unregistered_module_kind_is_rejected(oracle):
    class Doubler(nn.Module):
        def forward(self, x):
            return x * 2.0
    with pytest.raises(errors.FormatError):
        nn.serialize(nn.Sequential(Doubler(), nn.Linear(2, 2, backend=oracle.name)))


@pytest.mark.gpu
def test_reference_checkpoint_on_device_byte_identical_and_resumes(tmp_path):
    """The reference's CPU checkpoint loads onto the B200, writes back the same bytes, and
    the resumed step matches the oracle's resumed step."""
    be = gpu_backend()
    ck, opt, again = _resave(be, tmp_path)
    assert again == _gold()
    r = np.random.default_rng(5)
    x = r.standard_normal((6, 1, 12, 12)).astype(np.float32)
    y = r.integers(0, 10, 6).astype(np.int64)
    ck.model[5].p = 0.0  # no dropout draw: the two backends then run the same arithmetic
    loss_gpu = training.train_step(ck.model, x, y, opt)[0]
    ref = OracleBackend(name="ckpt-resume-oracle")
    registry.register(ref)
    try:
        ck2 = training.load_checkpoint(GOLD, backend=ref.name)
        opt2 = ck2.restore_optimizer()
        ck2.model[5].p = 0.0
        loss_ref = training.train_step(ck2.model, x, y, opt2)[0]
    finally:
        registry.unregister(ref.name)
    assert abs(loss_gpu - loss_ref) <= 1e-5 * max(abs(loss_ref), 1.0), (loss_gpu, loss_ref)
