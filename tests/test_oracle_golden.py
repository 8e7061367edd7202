"""Pin the numpy oracle (oracle/) to the reference's own outputs (tests/golden/)."""

import numpy as np
import pytest

from golden_util import check_against, op_cases, rng_arrays
from oracle import rng as orng
from oracle.kernels import KERNELS
from paper_2201_12465_b200 import errors, infer
from paper_2201_12465_b200.registry import OpCall

CASES = op_cases()


@pytest.mark.parametrize("case", CASES, ids=[c["id"] for c in CASES])
def test_oracle_matches_reference(case):
    shapes = [(np.shape(a), a.dtype) for a in case["input_arrays"]]
    from paper_2201_12465_b200 import dtypes
    from paper_2201_12465_b200.shape import Shape
    ins = [(Shape(s), dtypes.from_numpy(d)) for s, d in shapes]
    if "error" in case:
        with pytest.raises((errors.Error, ValueError, OverflowError)) as ei:
            shape, dt = infer.plan(case["name"], case["params"], ins)
            KERNELS[case["name"]](OpCall(case["name"], case["params"], shape, dt), case["input_arrays"])
        assert type(ei.value).__name__ == case["error"]
        return
    shape, dt = infer.plan(case["name"], case["params"], ins)
    assert list(shape) == case["shape"] and dt.name == case["dtype"]
    got = KERNELS[case["name"]](OpCall(case["name"], case["params"], shape, dt), case["input_arrays"])
    check_against(case, np.asarray(got), tol=1e-12 if case["name"] != "rand_normal" else 1e-15)


def test_rng_streams_bit_exact():
    g = rng_arrays()
    for k in range(5):
        seed, off, n = (int(v) for v in g[f"meta{k}"])
        assert np.array_equal(orng.words(seed, off, n), g[f"w{k}"])
        assert np.array_equal(orng.uniform(seed, off, n), g[f"u{k}"])
        assert np.allclose(orng.normal(seed, off, n), g[f"n{k}"], rtol=0, atol=1e-15)
