"""Extent allocator of the HBM block pool / host arena (CPU-only)."""

import random

import pytest

from paper_2601_10729_b200.kvpool import ExtentAllocator, PoolExhausted


def test_first_fit_and_coalescing():
    a = ExtentAllocator(100)
    x = a.alloc(30)
    y = a.alloc(30)
    z = a.alloc(40)
    assert (x, y, z) == (0, 30, 60) and a.free_blocks == 0
    with pytest.raises(PoolExhausted):
        a.alloc(1)
    a.release(y, 30)
    assert a.alloc(10) == 30          # first fit reuses the hole
    a.release(30, 10)
    a.release(x, 30)
    a.release(z, 40)
    assert a.free_blocks == 100 and a.alloc(100) == 0   # fully coalesced


def test_double_free_and_bounds():
    a = ExtentAllocator(10)
    s = a.alloc(4)
    a.release(s, 4)
    with pytest.raises(ValueError):
        a.release(s, 4)
    with pytest.raises(ValueError):
        a.release(8, 4)


def test_random_alloc_release_invariants():
    rng = random.Random(7)
    a = ExtentAllocator(1000)
    live = {}
    for _ in range(3000):
        if live and rng.random() < 0.45:
            start = rng.choice(sorted(live))
            a.release(start, live.pop(start))
        else:
            n = rng.randint(1, 60)
            try:
                start = a.alloc(n)
            except PoolExhausted:
                continue
            for s2, n2 in live.items():           # no overlap with live extents
                assert start + n <= s2 or s2 + n2 <= start
            live[start] = n
        assert a.in_use == sum(live.values())
    for start, n in list(live.items()):
        a.release(start, n)
    assert a.free_blocks == 1000 and a.alloc(1000) == 0
