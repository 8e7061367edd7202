"""The C++ caching allocator (simulate mode, no device) reproduces the reference
allocator's known answers: policies, counters, fragmentation, replay of the reference's
own synthetic trace (tests/golden/alloc.json, made by running minml.memory)."""

import pytest

from golden_util import alloc_meta, trace_lines
from paper_2201_12465_b200 import memory
from paper_2201_12465_b200.errors import AllocError, ManagerBusy, OutOfMemory

KIB, MIB = 1024, 1 << 20


def replay(lines, policy, threshold=None):
    m = memory.make_manager(policy, threshold=threshold, simulate=True)
    live, timeline = {}, []
    for line in lines:
        parts = line.split()
        if parts[0] == "A":
            live[parts[1]] = m.alloc(int(parts[2]), op=parts[3] if len(parts) > 3 else None)
        else:
            m.free(live.pop(parts[1]))
        timeline.append(m.stats().live_bytes_requested)
    return m, timeline


def test_caching_reuse_and_counters():
    m = memory.CachingManager(simulate=True)
    a = m.alloc(1000)
    assert a.granted_bytes == 1024 and a.internal_fragmentation == 24
    m.free(a)
    assert m.stats().cache_bytes == 1024
    b = m.alloc(900)
    assert b.granted_bytes == 1024 and m.stats().alloc_count == 1 and m.stats().cache_bytes == 0
    m.free(b)


def test_split_policies():
    m = memory.SplitRestrictedManager(threshold=MIB, simulate=True)
    big = m.alloc(512 * KIB)
    m.free(big)
    small = m.alloc(100 * KIB)
    assert small.granted_bytes == memory.round_up(100 * KIB)
    assert m.stats().cache_bytes == 512 * KIB - small.granted_bytes
    m.free(small)
    m = memory.SplitRestrictedManager(threshold=MIB, simulate=True)
    a = m.alloc(1024)
    m.free(a)
    b = m.alloc(700)
    assert b.granted_bytes == 1024 and m.stats().cache_bytes == 0
    m = memory.SplitRestrictedManager(threshold=MIB, simulate=True)
    big = m.alloc(2 * MIB)
    m.free(big)
    small = m.alloc(100 * KIB)
    assert small.granted_bytes == memory.bin_size(100 * KIB)
    assert m.stats().cache_bytes == memory.bin_size(2 * MIB)


def test_double_free_capacity_and_close():
    m = memory.NativeManager(simulate=True)
    b = m.alloc(64)
    assert b.granted_bytes == 64
    m.free(b)
    with pytest.raises(AllocError):
        m.free(b)
    c = memory.CachingManager(capacity=4096, simulate=True)
    a = c.alloc(2048)
    with pytest.raises(OutOfMemory):
        c.alloc(4096)
    with pytest.raises(ManagerBusy):
        c.close()
    c.free(a)
    c.close()
    s = c.stats()
    assert s.live_bytes_requested == 0 and s.cache_bytes == 0 and s.alloc_count == s.free_count


@pytest.mark.parametrize("key", sorted(alloc_meta()["replays"]))
def test_replay_matches_reference(key):
    want = alloc_meta()["replays"][key]
    label, policy, th = key.split("/")
    th = None if th == "None" else int(th)
    lines = trace_lines() if label == "bundled" else ["A 1 1000 conv", "A 2 600 bias", "F 1", "A 3 900 act",
                                                     "F 2", "F 3"]
    m, timeline = replay(lines, policy, th)
    assert m.peak_internal_fragmentation == want["peak_internal_fragmentation"]
    got = m.stats().as_dict()
    for k, v in want["stats"].items():
        assert got[k] == pytest.approx(v), (k, got[k], v)
    if want["live_req"] is not None:
        assert timeline == want["live_req"]


def test_split_cuts_fragmentation_20pct():
    lines = trace_lines()
    c, _ = replay(lines, "caching")
    s, _ = replay(lines, "split_restricted", 1 << 20)
    assert 1 - s.peak_internal_fragmentation / c.peak_internal_fragmentation >= 0.20
