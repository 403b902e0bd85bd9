"""In-step K1 kernel / plan per shape (attention-only steps, all layers resident).

Times all-resident decode steps (as tools/small_step_probe.py) with the in-step
choice pinned through OFB_K1_INSTEP (read at every launch):
  auto     the shipped policy
  split    split kernel, cost-model plan (wide when the grid is one wave)
  bal      split kernel, narrow, one CTA per SM less one SM per (request, KV head)
  cluster  cluster kernel (DSMEM combine)
The split kernel's consumers wait for the previous layer only before their
global writes (kv_ready 1 = late wait), so consecutive layers overlap.

    python tools/k1_instep_sweep.py [--batches 1,2,4,8,16] [--contexts 1024,...] [--max-tokens 262144]
"""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_10729_b200.core import PlacementMatrix, RequestState  # noqa: E402
from paper_2601_10729_b200.executor import B200Executor, ModelShape  # noqa: E402


def _arg(flag, default):
    return [int(v) for v in sys.argv[sys.argv.index(flag) + 1].split(",")] if flag in sys.argv else default


MODES = os.environ.get("SWEEP_MODES", "auto,split,bal,cluster").split(",")
max_tokens = _arg("--max-tokens", [262144])[0]
shapes = {"8B": ModelShape(32, 32, 8), "70B-TP8-shard": ModelShape(32, 8, 1)}
if os.environ.get("SWEEP_SHAPES"):
    shapes = {k: v for k, v in shapes.items() if k in os.environ["SWEEP_SHAPES"].split(",")}
for name, shape in shapes.items():
    for B in _arg("--batches", (1, 2, 4, 8, 16)):
        for ctx in _arg("--contexts", (1024, 4096, 8192, 16384, 32768, 65536)):
            if B * ctx > max_tokens:
                continue
            cap = -(-(ctx + 64 + 1) // 16)
            nblk = -(-(ctx + 1) // 16)
            batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=ctx, target_output_tokens=64)
                     for i in range(B)]
            pm = PlacementMatrix.from_strides(range(B), 32, [None] * B)
            ex = B200Executor(shape, device_blocks=B * 32 * cap + 16, host_blocks=16, fill="zeros")
            ex.install(batch, pm)
            inp = ex.synthetic_inputs(B, step=0)
            kv = B * 32 * nblk * shape.num_kv_heads * 16 * 128 * 2 * 2
            row = {"shape": name, "B": B, "context": ctx}
            for mode in MODES:
                if mode == "auto":
                    os.environ.pop("OFB_K1_INSTEP", None)
                else:
                    os.environ["OFB_K1_INSTEP"] = mode
                for _ in range(5):
                    ex.decode_step(batch, None, inp, sync=False)
                ex.drain()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(40):
                    ex.decode_step(batch, None, inp, sync=False)
                e1.record()
                ex.drain()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 40
                row[mode] = round(ms * 1e3 / 32, 2)
            os.environ.pop("OFB_K1_INSTEP", None)
            row["roofline_us"] = round(kv / 32 / 6.45e12 * 1e6, 2)
            print(json.dumps(row), flush=True)
            ex.close()
