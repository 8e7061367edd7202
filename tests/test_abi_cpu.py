"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every symbol
include/paper_b200.h declares, and its host-only entry points behave."""

import os
import re

from paper_2201_12465_b200.gpu import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    with open(os.path.join(ROOT, "include", "paper_b200.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(pb_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _declared()
    assert len(declared) >= 40
    missing = [n for n in declared if not hasattr(lib, n)]
    assert not missing, missing
    assert set(declared) == set(_lib.SIGNATURES), set(declared) ^ set(_lib.SIGNATURES)


def test_device_count_does_not_crash():
    assert _lib.load().pb_device_count() >= 0


def test_bin_and_round_helpers_match_reference_known_answers():
    from golden_util import alloc_meta
    lib = _lib.load()
    meta = alloc_meta()
    for n, want in meta["bin_size"].items():
        assert lib.pb_bin_size(int(n)) == want
    for n, want in meta["round_up"].items():
        assert lib.pb_round_up(int(n)) == want


def test_tensor_descriptor_layout():
    assert _lib.TENSOR.size == 144 and _lib.SCALAR.size == 24 and _lib.CONV.size == 16
    vals = _lib.TENSOR.unpack(_lib.pack_tensor(0x1000, 4, (2, 3), (3, 1)))
    assert vals[:3] == (0x1000, 4, 2) and vals[3:5] == (2, 3) and vals[11:13] == (3, 1)
