"""K1 split length inside an all-resident decode step (B=1, the cfg3 regime): per
context, the per-layer cost at each blocks-per-split (OFB_K1_BPS, read per launch)
against the cost model's pick, on one executor per context.

    python tools/k1_bps_step.py [--shape 8B|70B-TP8-shard] [--batch 1] [--contexts 8192,...]
"""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_10729_b200 import _native  # noqa: E402
from paper_2601_10729_b200.core import PlacementMatrix, RequestState  # noqa: E402
from paper_2601_10729_b200.executor import B200Executor, ModelShape  # noqa: E402


def _arg(flag, default, cast=int):
    return [cast(v) for v in sys.argv[sys.argv.index(flag) + 1].split(",")] if flag in sys.argv else default


shape_name = _arg("--shape", ["8B"], str)[0]
shape = {"8B": ModelShape(32, 32, 8), "70B-TP8-shard": ModelShape(32, 8, 1)}[shape_name]
B = _arg("--batch", [1])[0]
lib = _native.load()


def step_us(ex, batch, inp, iters=30):
    for _ in range(4):
        ex.decode_step(batch, None, inp, sync=False)
    ex.drain()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        ex.decode_step(batch, None, inp, sync=False)
    e1.record()
    ex.drain()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3 / shape.num_layers


for ctx in _arg("--contexts", [8192, 16384, 32768, 65536, 131072]):
    cap = -(-(ctx + 64 + 1) // 16)
    batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=ctx, target_output_tokens=64) for i in range(B)]
    pm = PlacementMatrix.from_strides(range(B), shape.num_layers, [None] * B)
    ex = B200Executor(shape, device_blocks=B * shape.num_layers * cap + 16, host_blocks=16, fill="zeros")
    ex.install(batch, pm)
    inp = ex.synthetic_inputs(B, step=0)
    nblk = -(-(ctx + 1) // 16)
    pairs = B * shape.num_kv_heads
    cands = sorted({b for b in (8, 16, 32, 64, 128, 256) if b <= max(nblk, 8)} |
                   {-(-nblk // (t // pairs)) for t in (148, 296, 444) if t // pairs >= 1})
    os.environ.pop("OFB_K1_BPS", None)
    row = {"shape": shape_name, "B": B, "context": ctx, "auto": round(step_us(ex, batch, inp), 2)}
    for b in cands:
        if b > 256:
            continue
        os.environ["OFB_K1_BPS"] = str(b)
        row[f"bps{b}"] = round(step_us(ex, batch, inp), 2)
        row[f"ctas{b}"] = pairs * -(-nblk // b)
    os.environ.pop("OFB_K1_BPS", None)
    print(json.dumps(row), flush=True)
    ex.close()
