"""Per-launch floor of K1 in a graph-replayed PDL chain: tiny contexts (one
block per request), so the time is launch + prologue + one tile + merge /
combine, not bandwidth.  Also a do-nothing kernel chain for the bare launch cost.

    python tools/k1_floor.py
"""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_10729_b200 import ops  # noqa: E402

dev = torch.device("cuda:0")


def graph_us(fn, iters=32):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / iters * 1e3)
    return statistics.median(ts)


x = torch.zeros(1, device=dev)
rows = {"torch_add_chain_us": graph_us(lambda: x.add_(1.0))}
for hq, hkv, seq in [(8, 1, 16), (8, 1, 256), (32, 8, 16), (32, 8, 256)]:
    pool = torch.randn((64, hkv, 2, 16, 128), device=dev).to(torch.bfloat16)
    bt = torch.arange(16, dtype=torch.int32, device=dev).reshape(1, 16)
    lens = torch.full((1,), seq, dtype=torch.int32, device=dev)
    q = torch.randn((1, hq, 128), device=dev).to(torch.bfloat16)
    out = torch.empty_like(q)
    ws = ops.workspace(1, hq, hkv, 256, dev)
    for v in ("split", "cluster"):
        ops.set_attention_kernel(v)
        rows[f"{v} hq={hq} hkv={hkv} seq={seq}"] = graph_us(
            lambda: ops.decode_attention(q, pool, bt, lens, out=out, max_seq_len=seq, ws=ws))
ops.set_attention_kernel("auto")
print(json.dumps(rows, indent=1))
