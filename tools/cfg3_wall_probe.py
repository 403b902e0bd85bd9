"""Where cfg3's wall clock goes beyond the GPU time in live-wall mode: per-step
(wall - device) distribution of the serving loop, with Python's cyclic GC on
(default) and frozen (``gc.freeze()`` after setup + ``gc.disable()`` for the run).

    python tools/cfg3_wall_probe.py [--requests 24]
"""
import argparse
import gc
import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def run(a, freeze):
    args = argparse.Namespace(cfg3_rate=30.0, cfg3_requests=a.requests, cfg3_output_median=256,
                              cfg3_budget_blocks=655360, cfg3_calibrate=False, slo_scale=1.5)
    from paper_2601_10729_b200.engine import Simulation
    from paper_2601_10729_b200.executor import B200Executor, LLAMA31_8B
    from paper_2601_10729_b200.policies import PolicyKind, make_policy

    trace, profile, slo, cfg = bench.cfg3_setup(args)
    ex = B200Executor.for_trace(trace, profile, shape=LLAMA31_8B, max_batch=cfg.max_batch)
    policy = make_policy(PolicyKind.ORBIT, profile, slo, max_batch=cfg.max_batch,
                         token_cap=cfg.batch_token_cap)
    sim = Simulation(trace, policy, profile, slo, cfg, executor=ex, mode="live-wall")
    if freeze:
        gc.collect()
        gc.freeze()
        gc.disable()
    t0 = time.perf_counter()
    log = sim.execute()
    wall = time.perf_counter() - t0
    if freeze:
        gc.enable()
        gc.unfreeze()
    steps = [r for r in log if r["kind"] == "step"]
    host = sorted((r["payload"]["wall_us"] - r["payload"]["measured_us"]) / 1e3 for r in steps)
    n = len(host)
    out = {"gc_frozen": freeze, "steps": n, "wall_s": round(wall, 3),
           "host_ms_median": round(statistics.median(host), 4),
           "host_ms_mean": round(sum(host) / n, 4),
           "host_ms_p90": round(host[int(0.9 * n)], 4), "host_ms_p99": round(host[int(0.99 * n)], 4),
           "host_ms_max": round(host[-1], 3),
           "host_ms_top20_sum": round(sum(host[-20:]), 2),
           "tokens_per_s_clock": round(sum(len(r["payload"].get("ids", [])) or 1 for r in steps)
                                       / (sum(r["payload"]["wall_us"] for r in steps) * 1e-6), 1)}
    ex.close()
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=24)
    a = ap.parse_args()
    for freeze in (False, True, False, True):
        print(json.dumps(run(a, freeze)), flush=True)
