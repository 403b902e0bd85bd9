"""The native exact solver (ofb_plan_solve) returns the same plans as the numpy
restatement (itself pinned to the reference by tests/test_golden.py and the
reference suite) on random instances, including batches past the reference's
tractable range.  CPU-only: the planner is host code."""

import random
import time

import pytest

from paper_2601_10729_b200 import planner
from paper_2601_10729_b200.core import PlacementMatrix, RequestState, SloConfig, SystemProfile
from paper_2601_10729_b200.latency import batch_decode_latency_fast


def _plan_sig(p):
    if isinstance(p, planner.Infeasible):
        return ("infeasible", p.reason)
    return (p.placement.rows, p.decode_window, p.expiry_step,
            p.predicted_latency.total_latency_ms.hex())


def _instance(rng, L, B):
    batch = [RequestState(id=r, arrival_time_ms=float(rng.randint(0, 3)),
                          prompt_tokens=rng.randint(10, 900), target_output_tokens=400)
             for r in range(B)]
    for r in batch:
        r.generated_tokens = rng.randint(0, 20)
        r.deposit_balance = rng.randint(0, 2)
        r.sync_blocks()
    total = sum(r.blocks_per_layer for r in batch) * L
    prof = SystemProfile(L, rng.choice([0.1, 0.3, 1.0]), rng.choice([0.0, 0.0003]),
                         rng.choice([3.0, 20.0, 80.0]),
                         max(max(r.blocks_per_layer for r in batch) + 2,
                             int(total * rng.uniform(0.3, 1.1))), 16)
    base = batch_decode_latency_fast(PlacementMatrix.all_resident([r.id for r in batch], L),
                                     batch, prof).total_latency_ms
    slo = SloConfig(base * rng.choice([1.0, 1.3, 2.0, 5.0]), base * 2,
                    violation_cap=rng.choice([0.5, 1.0, 2.0]), window_min=rng.randint(1, 4),
                    window_max=rng.randint(4, 12))
    paused = tuple(RequestState(id=50 + j, arrival_time_ms=0.0, prompt_tokens=rng.randint(10, 200),
                                target_output_tokens=100) for j in range(rng.choice([0, 1])))
    snap = None if rng.random() < 0.5 else {r.id: rng.uniform(0, 2) for r in [*batch, *paused]}
    return batch, prof, slo, paused, snap


def _both(fn):
    old = planner.SOLVER
    try:
        planner.SOLVER = "native"
        a = fn()
        planner.SOLVER = "python"
        b = fn()
    finally:
        planner.SOLVER = old
    return a, b


@pytest.mark.parametrize("L,B,count", [(4, 4, 60), (9, 3, 60), (12, 3, 40), (32, 3, 25), (32, 4, 6)])
def test_native_matches_numpy(L, B, count):
    rng = random.Random(L * 100 + B)
    for _ in range(count):
        batch, prof, slo, paused, snap = _instance(rng, L, B)
        step = rng.randint(1, 30)
        a, b = _both(lambda: planner.solve(batch, prof, slo, step, paused=paused,
                                           deposit_snapshot=snap))
        assert _plan_sig(a) == _plan_sig(b)
        a, b = _both(lambda: planner.solve_capacity_only(batch, prof, slo, step))
        assert _plan_sig(a) == _plan_sig(b)
        a, b = _both(lambda: planner.solve_one_step_ahead(batch, prof, slo, step, paused=paused,
                                                          deposit_snapshot=snap))
        assert _plan_sig(a) == _plan_sig(b)


def test_native_is_faster_at_b5():
    rng = random.Random(5)
    batch, prof, slo, paused, snap = _instance(rng, 32, 5)
    t0 = time.perf_counter()
    planner.SOLVER = "native"
    a = planner.solve(batch, prof, slo, 1, paused=paused, deposit_snapshot=snap)
    t_native = time.perf_counter() - t0
    planner.SOLVER = "python"
    t0 = time.perf_counter()
    b = planner.solve(batch, prof, slo, 1, paused=paused, deposit_snapshot=snap)
    t_py = time.perf_counter() - t0
    planner.SOLVER = "native"
    assert _plan_sig(a) == _plan_sig(b)
    assert t_native < t_py


@pytest.mark.gpu
@pytest.mark.parametrize("L,B,count", [(4, 4, 30), (9, 3, 30), (32, 4, 6), (32, 5, 3)])
def test_gpu_enumeration_matches_host(L, B, count):
    """SOLVER="native-gpu" (candidate space enumerated + radix-sorted on the GPU)
    returns exactly the host solver's plans, windows and latencies."""
    rng = random.Random(1000 + L * 10 + B)
    for _ in range(count):
        batch, prof, slo, paused, snap = _instance(rng, L, B)
        for cap_only in (False, True):
            def run():
                if cap_only:
                    return _plan_sig(planner.solve_capacity_only(batch, prof, slo, 3))
                return _plan_sig(planner.solve(batch, prof, slo, 3, paused=paused,
                                               deposit_snapshot=snap))
            old = planner.SOLVER
            try:
                planner.SOLVER = "native"
                a = run()
                planner.SOLVER = "native-gpu"
                b = run()
            finally:
                planner.SOLVER = old
            assert a == b


@pytest.mark.gpu
def test_gpu_enumeration_b8_l32():
    """B=8 at L=32 (214 M candidates; the reference is intractable here): the GPU
    enumeration returns the host solver's plan, much faster."""
    from paper_2601_10729_b200 import defaults
    from paper_2601_10729_b200.calibrate import b200_profile

    rng = random.Random(8)
    prof = b200_profile(32, 8, gpu_block_budget=60000 * 8 // 4)
    batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=rng.randint(2000, 30000),
                          target_output_tokens=64) for i in range(8)]
    slo = defaults.default_slo(prof, 60.0)
    old = planner.SOLVER
    try:
        planner.SOLVER = "native"
        t = time.perf_counter()
        a = _plan_sig(planner.solve(batch, prof, slo, 1))
        t_host = time.perf_counter() - t
        planner.SOLVER = "native-gpu"
        planner.solve(batch, prof, slo, 1)            # warm-up (context, cub)
        t = time.perf_counter()
        b = _plan_sig(planner.solve(batch, prof, slo, 1))
        t_gpu = time.perf_counter() - t
    finally:
        planner.SOLVER = old
    assert a == b
    assert t_gpu < t_host, (t_gpu, t_host)


@pytest.mark.gpu
@pytest.mark.parametrize("window,shapes", [(5, ((4, 4), (9, 3))),
                                           (300, ((4, 4), (9, 3), (12, 4), (32, 4), (32, 5))),
                                           (5000, ((4, 4), (9, 3), (12, 4), (32, 4), (32, 5)))])
def test_gpu_enumeration_windows_match_host(window, shapes, monkeypatch):
    """The GPU candidate list is served in bounded windows (whole lower-bound
    keys, or index ranges of one oversized key): forcing tiny windows changes
    nothing in the plans, windows and latencies."""
    monkeypatch.setenv("OFB_PLAN_WINDOW", str(window))
    rng = random.Random(4242 + window)
    multi = 0
    for L, B in shapes:
        for _ in range(4):
            batch, prof, slo, paused, snap = _instance(rng, L, B)
            for cap_only in (False, True):
                def run():
                    if cap_only:
                        return _plan_sig(planner.solve_capacity_only(batch, prof, slo, 3))
                    return _plan_sig(planner.solve(batch, prof, slo, 3, paused=paused,
                                                   deposit_snapshot=snap))
                old = planner.SOLVER
                try:
                    planner.SOLVER = "native"
                    a = run()
                    planner.SOLVER = "native-gpu"
                    b = run()
                    multi += (planner.LAST_NATIVE_STATS or {}).get("windows", 0) > 1
                finally:
                    planner.SOLVER = old
                assert a == b
    assert multi > 0


@pytest.mark.gpu
@pytest.mark.parametrize("L,B", [(4, 9), (4, 10)])
def test_gpu_enumeration_past_b8_matches_numpy(L, B, monkeypatch):
    """Batches past the host solver's range (B = 9-10) against the numpy
    restatement, with small windows so several are materialised."""
    monkeypatch.setenv("OFB_PLAN_WINDOW", "20000")
    rng = random.Random(9000 + L * 10 + B)
    for _ in range(2):
        batch, prof, slo, paused, snap = _instance(rng, L, B)
        old = planner.SOLVER
        try:
            planner.SOLVER = "native-gpu"
            a = _plan_sig(planner.solve(batch, prof, slo, 2, paused=paused, deposit_snapshot=snap))
            c = _plan_sig(planner.solve_capacity_only(batch, prof, slo, 2))
            planner.SOLVER = "python"
            b = _plan_sig(planner.solve(batch, prof, slo, 2, paused=paused, deposit_snapshot=snap))
            d = _plan_sig(planner.solve_capacity_only(batch, prof, slo, 2))
        finally:
            planner.SOLVER = old
        assert a == b
        assert c == d


@pytest.mark.gpu
def test_gpu_enumeration_b9_l32_matches_host(monkeypatch):
    """B = 9 at L = 32 (2.36 G candidates, past the 2^32 index of the previous
    composite key): the windowed GPU enumeration equals the host DFS run past
    its default range."""
    from paper_2601_10729_b200 import defaults
    from paper_2601_10729_b200.calibrate import b200_profile

    monkeypatch.setenv("OFB_PLAN_HOST_SPACE_LOG2", "32")
    monkeypatch.setattr(planner, "_NATIVE_MAX_SPACE", 1 << 32)
    rng = random.Random(9)
    prof = b200_profile(32, 8, gpu_block_budget=60000 * 9 // 4)
    batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=rng.randint(2000, 30000),
                          target_output_tokens=64) for i in range(9)]
    slo = defaults.default_slo(prof, 60.0)
    old = planner.SOLVER
    try:
        planner.SOLVER = "native-gpu"
        b = _plan_sig(planner.solve(batch, prof, slo, 1))
        stats = dict(planner.LAST_NATIVE_STATS)
        planner.SOLVER = "native"
        a = _plan_sig(planner.solve(batch, prof, slo, 1))
    finally:
        planner.SOLVER = old
    assert stats["feasible"] > 0
    assert a == b
