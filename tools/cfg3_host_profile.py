"""Where cfg3's host control goes in live-wall mode: the serving loop (the
reference kvsim engine + the B200 executor seam) under cProfile, on a B200.
Prints the top functions by cumulative and by own time.

    python tools/cfg3_host_profile.py [--requests 8] [--mode live-wall]
"""
import argparse
import cProfile
import io
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=8)
    ap.add_argument("--mode", default="live-wall")
    ap.add_argument("--top", type=int, default=45)
    a = ap.parse_args()
    args = argparse.Namespace(cfg3_rate=30.0, cfg3_requests=a.requests, cfg3_output_median=256,
                              cfg3_budget_blocks=655360, cfg3_calibrate=False, slo_scale=1.5)
    from paper_2601_10729_b200.engine import Simulation
    from paper_2601_10729_b200.executor import B200Executor, LLAMA31_8B
    from paper_2601_10729_b200.policies import PolicyKind, make_policy

    trace, profile, slo, cfg = bench.cfg3_setup(args)
    ex = B200Executor.for_trace(trace, profile, shape=LLAMA31_8B, max_batch=cfg.max_batch)
    policy = make_policy(PolicyKind.ORBIT, profile, slo, max_batch=cfg.max_batch,
                         token_cap=cfg.batch_token_cap)
    sim = Simulation(trace, policy, profile, slo, cfg, executor=ex, mode=a.mode)
    prof = cProfile.Profile()
    t0 = time.perf_counter()
    prof.enable()
    log = sim.execute()
    prof.disable()
    wall = time.perf_counter() - t0
    steps = [r for r in log if r["kind"] == "step"]
    gpu_ms = sum(r["payload"]["measured_us"] for r in steps) / 1e3
    print(f"steps {len(steps)}  wall {wall:.2f} s  gpu {gpu_ms / 1e3:.2f} s  "
          f"host+sync per step {(wall * 1e3 - gpu_ms) / max(1, len(steps)):.3f} ms (profiled)")
    for key in ("cumulative", "tottime"):
        s = io.StringIO()
        pstats.Stats(prof, stream=s).sort_stats(key).print_stats(a.top)
        print(s.getvalue())
    ex.close()


if __name__ == "__main__":
    main()
