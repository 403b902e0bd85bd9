"""Whole-decoder TP step (tp.TensorParallelLlama) at a TP-N shard shape on one GPU:
device ms per step (CUDA events, back-to-back steps) and, run under
``ncu --metrics gpu__time_duration.sum``, the per-kernel launch list of the
non-attention work (projections, norms, activations, K6).

  python tools/decoder_probe.py --tp 8 --prompt 4096 --steps 6 [--c1 k6|nccl]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2601_10729_b200.core import PlacementMatrix, RequestState  # noqa: E402
from paper_2601_10729_b200.executor import B200Executor, ModelShape  # noqa: E402
from paper_2601_10729_b200.tp import HeadShard, TensorParallelLlama  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tp", type=int, default=8)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--prompt", type=int, default=4088)
    ap.add_argument("--layers", type=int, default=80)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--c1", default="k6")
    ap.add_argument("--host-profile", action="store_true",
                    help="cProfile one step's host-side enqueue (top functions)")
    ap.add_argument("--profile-last", action="store_true",
                    help="cudaProfilerStart/Stop around the last step (ncu --profile-from-start off)")
    args = ap.parse_args()
    shard = HeadShard(0, args.tp, 64, 8)
    shape = ModelShape(args.layers, shard.local_q, shard.local_kv)
    B, L = args.batch, args.layers
    cap = -(-(args.prompt + args.steps + 8) // 16)
    ex = B200Executor(shape, device_blocks=L * B * cap + 2 * B * cap + 64, host_blocks=64,
                      staging_slots=2, fill="zeros")
    batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=args.prompt,
                          target_output_tokens=args.steps + 4) for i in range(B)]
    ex.install(batch, PlacementMatrix.from_strides([r.id for r in batch], L, [None] * B))
    dec = TensorParallelLlama(ex, shard, 8192, 28672, c1=args.c1, max_batch=B)
    x = torch.randn((B, 8192), device=ex.device).to(torch.bfloat16)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    torch.cuda.synchronize()
    evs[0].record()
    import time
    host_ms = []
    for i in range(args.steps):
        if args.profile_last and i == args.steps - 1:
            torch.cuda.synchronize()
            torch.cuda.profiler.start()
        t0 = time.perf_counter()
        if args.host_profile and i == args.steps - 1:
            import cProfile
            import pstats
            prof = cProfile.Profile()
            prof.enable()
            dec.step(batch, x)
            prof.disable()
            pstats.Stats(prof).sort_stats("tottime").print_stats(15)
        else:
            dec.step(batch, x)
        host_ms.append((time.perf_counter() - t0) * 1e3)
        if args.profile_last and i == args.steps - 1:
            torch.cuda.synchronize()
            torch.cuda.profiler.stop()
        evs[i + 1].record()
        for r in batch:
            r.record_generated_token()
    torch.cuda.synchronize()
    ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    print(json.dumps({"tp": args.tp, "batch": B, "prompt": args.prompt, "c1": args.c1,
                      "weight_bytes": dec.weight_bytes, "step_ms": ms, "host_enqueue_ms": host_ms}))
    dec.close()
    ex.close()


if __name__ == "__main__":
    main()
