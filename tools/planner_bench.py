"""Exact-solve latency: reference kvsim (if importable) vs this package's numpy
restatement vs the native solver (host DFS, GPU enumeration), on a
B200-calibrated 8B profile (L=32).  Every plan is compared for bit-identity.

    python tools/planner_bench.py [--max-batch 10] [--host-max 8]

B = 9-10 (2.4 G / 26 G candidates) run on the GPU enumeration only, unless
--host-max raises the host DFS's range (OFB_PLAN_HOST_SPACE_LOG2, needs memory).
"""
import argparse
import json
import random
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_10729_b200 import _native, defaults, planner  # noqa: E402
from paper_2601_10729_b200.calibrate import b200_profile  # noqa: E402
from paper_2601_10729_b200.core import RequestState  # noqa: E402

_native.load()
REF = None
if Path("/root/reference/pkg/src").exists():
    sys.path.insert(0, "/root/reference/pkg/src")
    import kvsim as REF  # noqa: E402


def sig(p):
    if not hasattr(p, "placement"):
        return ("infeasible", p.reason)
    return ([list(r) for r in p.placement.rows], p.decode_window, p.expiry_step,
            p.predicted_latency.total_latency_ms.hex())


ap = argparse.ArgumentParser()
ap.add_argument("--max-batch", type=int, default=8)
ap.add_argument("--min-batch", type=int, default=1)
ap.add_argument("--host-max", type=int, default=8)
args = ap.parse_args()
if args.host_max > 8:
    import os

    os.environ["OFB_PLAN_HOST_SPACE_LOG2"] = "36"
    planner._NATIVE_MAX_SPACE = 1 << 36

rows = []
for B in range(args.min_batch, args.max_batch + 1):
    rng = random.Random(B)
    prof = b200_profile(32, 8, gpu_block_budget=60000 * B // 4)
    batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=rng.randint(2000, 30000),
                          target_output_tokens=64) for i in range(B)]
    slo = defaults.default_slo(prof, 60.0)
    rec = {"batch": B}
    p_nat = None
    if B <= args.host_max:
        planner.SOLVER = "native"
        t = time.perf_counter(); p_nat = planner.solve(batch, prof, slo, 1)
        rec["native_ms"] = (time.perf_counter() - t) * 1e3
        rec["plan"] = sig(p_nat)[0] if sig(p_nat)[0] == "infeasible" else [r.count(0) for r in p_nat.placement.rows]
        rec["native_stats"] = planner.LAST_NATIVE_STATS
    try:
        import torch

        if torch.cuda.is_available():
            planner.SOLVER = "native-gpu"
            planner.solve(batch, prof, slo, 1)             # warm-up (context, cub)
            t = time.perf_counter(); p_gpu = planner.solve(batch, prof, slo, 1)
            rec["native_gpu_ms"] = (time.perf_counter() - t) * 1e3
            rec["native_gpu_stats"] = planner.LAST_NATIVE_STATS
            if p_nat is not None:
                rec["native_gpu_equal"] = sig(p_gpu) == sig(p_nat)
            else:
                rec["plan"] = (sig(p_gpu)[0] if sig(p_gpu)[0] == "infeasible"
                               else [r.count(0) for r in p_gpu.placement.rows])
            planner.SOLVER = "native"
    except ImportError:
        pass
    if B <= 6:
        planner.SOLVER = "python"
        t = time.perf_counter(); p_py = planner.solve(batch, prof, slo, 1)
        rec["numpy_ms"] = (time.perf_counter() - t) * 1e3
        rec["numpy_equal"] = sig(p_py) == sig(p_nat)
    if REF is not None and B <= 6:
        rprof = REF.SystemProfile(**{k: getattr(prof, k) for k in prof.__dataclass_fields__})
        rslo = REF.SloConfig(**{k: getattr(slo, k) for k in slo.__dataclass_fields__})
        rb = [REF.RequestState(id=r.id, arrival_time_ms=0.0, prompt_tokens=r.prompt_tokens,
                               target_output_tokens=64) for r in batch]
        t = time.perf_counter(); p_ref = REF.solve(rb, rprof, rslo, 1)
        rec["reference_ms"] = (time.perf_counter() - t) * 1e3
        rec["reference_equal"] = sig(p_ref) == sig(p_nat)
    rows.append(rec)
    print(json.dumps(rec), flush=True)
planner.SOLVER = "native"
