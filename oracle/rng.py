"""splitmix64 counter stream, restated from minml/rng.py:16-51 (test oracle)."""

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def words(seed, offset, count):
    """uint64 words for counters offset..offset+count-1 (minml/rng.py:28-33)."""
    i = np.arange(offset, offset + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & ((1 << 64) - 1)) + (i + np.uint64(1)) * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def uniform(seed, offset, count):
    """53-bit doubles in [0,1) (minml/rng.py:36-38)."""
    return (words(seed, offset, count) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def normal(seed, offset, count):
    """Box-Muller, pairs interleaved cos/sin (minml/rng.py:41-51)."""
    half = (count + 1) // 2
    u1 = uniform(seed, offset, half)
    u2 = uniform(seed, offset + half, half)
    rad = np.sqrt(-2.0 * np.log1p(-u1))
    ang = 2.0 * np.pi * u2
    out = np.stack([rad * np.cos(ang), rad * np.sin(ang)], axis=1).reshape(-1)
    return out[:count]
