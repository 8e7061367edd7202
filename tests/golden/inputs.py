"""Deterministic synthetic batches shared by the golden generator and the parity tests
(PCG64 streams are stable across numpy versions, so only seeds are committed)."""

import zlib

import numpy as np


def batch(name, k, shape, classes, batch_size, tokens=None):
    rng = np.random.default_rng(zlib.crc32(f"{name}/{k}".encode()))
    if tokens is not None:
        seq, vocab = tokens
        x = rng.integers(0, vocab, (batch_size, seq)).astype(np.int64)
    else:
        x = rng.standard_normal((batch_size,) + tuple(shape)).astype(np.float32)
    y = rng.integers(0, classes, batch_size).astype(np.int64)
    return x, y
