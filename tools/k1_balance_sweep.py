"""In-step K1 split length vs SM balance at B = 1..2 (the cfg3 regime).

The split plan's cost model (decode_attention.cu plan_splits) prices HBM and a
per-CTA stream rate but not how the grid lands on the 148 SMs: e.g. the 8B
shape at B=1, 16K runs 256 narrow CTAs (108 SMs hold two, 40 hold one).  This
probe times all-resident decode steps (as tools/small_step_probe.py) with the
split length pinned through OFB_K1_BPS (read at every launch) to grids of
one CTA per SM (wide kernel), two / three per SM (narrow), and the default.

    python tools/k1_balance_sweep.py [--contexts 8192,16384,32768,65536] [--batches 1,2]
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


SMS = torch.cuda.get_device_properties(0).multi_processor_count


def candidates(pairs, nblk):
    out = {"default": None}
    for per_sm in (1, 2, 3):
        ns = max(1, (SMS * per_sm) // pairs)
        bps = -(-nblk // ns)
        if bps <= 256:
            out[f"{per_sm}/SM"] = bps
    # one CTA per SM less one SM per pair: the pairs' combining CTAs keep theirs
    ns = max(1, (SMS - pairs) // pairs)
    bps = -(-nblk // ns)
    if bps <= 256:
        out["1/SM-c"] = bps
    return out


shapes = {"8B": ModelShape(32, 32, 8), "70B-TP8-shard": ModelShape(32, 8, 1)}
for name, shape in shapes.items():
    for B in _arg("--batches", (1, 2)):
        for ctx in _arg("--contexts", (8192, 16384, 32768, 65536)):
            cap = -(-(ctx + 64 + 1) // 16)
            nblk = -(-(ctx + 1) // 16)
            batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=ctx, target_output_tokens=64)
                     for i in range(B)]
            pm = PlacementMatrix.from_strides(range(B), 32, [None] * B)
            ex = B200Executor(shape, device_blocks=B * 32 * cap + 16, host_blocks=16, fill="zeros")
            ex.install(batch, pm)
            inp = ex.synthetic_inputs(B, step=0)
            for label, bps in candidates(B * shape.num_kv_heads, nblk).items():
                if bps is None:
                    os.environ.pop("OFB_K1_BPS", None)
                else:
                    os.environ["OFB_K1_BPS"] = str(bps)
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
                kv = B * 32 * nblk * shape.num_kv_heads * 16 * 128 * 2 * 2
                print(json.dumps({"shape": name, "B": B, "context": ctx, "plan": label, "bps": bps,
                                  "us_per_layer": round(ms * 1e3 / 32, 2),
                                  "hbm_gbs": round(kv / (ms * 1e-3) / 1e9, 1)}), flush=True)
            os.environ.pop("OFB_K1_BPS", None)
            ex.close()
