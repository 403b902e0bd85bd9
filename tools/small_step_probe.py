"""All-resident decode steps at small batch (the cfg3 regime): device time per
step for the 8B shape and the 70B TP8 rank shard (8 q / 1 KV head), B in {1, 4}
(--batches 1,2,4), 4K and 16K context (--contexts 1024,4096),
stream-launched and pipelined: the per-layer K1 cost inside
a step (K1 of a layer without a fetch streams its KV before the PDL wait).
Run once as is and once with OFB_PDL=0 to see what programmatic dependent launch
(+ kv_ready KV streaming before the wait) buys when each layer is short."""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_10729_b200.core import PlacementMatrix, RequestState  # noqa: E402
from paper_2601_10729_b200.executor import B200Executor, ModelShape  # noqa: E402

import itertools  # noqa: E402

def _arg(flag, default):
    return [int(v) for v in sys.argv[sys.argv.index(flag) + 1].split(",")] if flag in sys.argv else default


for (name, shape), B, ctx in itertools.product(
        [("8B", ModelShape(32, 32, 8)), ("70B-TP8-shard", ModelShape(32, 8, 1))],
        _arg("--batches", (1, 4)), _arg("--contexts", (4096, 16384))):
    cap = -(-(ctx + 64 + 1) // 16)
    batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=ctx, target_output_tokens=64)
             for i in range(B)]
    pm = PlacementMatrix.from_strides(range(B), 32, [None] * B)
    ex = B200Executor(shape, device_blocks=B * 32 * cap + 16, host_blocks=16, fill="zeros")
    ex.install(batch, pm)
    inp = ex.synthetic_inputs(B, step=0)
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
    print(json.dumps({"shape": name, "B": B, "context": ctx, "pdl": os.environ.get("OFB_PDL", "1"),
                      "ms_per_step": ms, "us_per_layer": ms * 1e3 / 32}), flush=True)
    ex.close()
