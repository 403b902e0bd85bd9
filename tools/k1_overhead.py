"""K1 fixed cost vs streaming rate: graph-replayed back-to-back launches over a
context sweep, so per-launch time = device time (no Python launch cost).

time(T) ~= fixed + bytes(T) / rate; the intercept is launch + ramp + drain +
combine, the slope the steady HBM read rate.

    python tools/k1_overhead.py --batch 32 --hq 8 --hkv 1 [--variant stream]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_10729_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--hq", type=int, default=8)
ap.add_argument("--hkv", type=int, default=1)
ap.add_argument("--seqs", default="16,1024,8192,32768,65536")
ap.add_argument("--variant", default="auto", choices=["stream", "split", "auto"])
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()

dev = torch.device("cuda:0")
ops.set_attention_kernel(a.variant)
for seq in [int(s) for s in a.seqs.split(",")]:
    nblk = (seq + 15) // 16
    layer_bytes = a.batch * nblk * a.hkv * 8192
    layers = max(2, min(16, (1 << 30) // max(layer_bytes, 1) + 1))
    pools = [torch.empty((a.batch * nblk, a.hkv, 2, 16, 128), dtype=torch.bfloat16, device=dev).normal_()
             for _ in range(layers)]
    bt = torch.arange(a.batch * nblk, dtype=torch.int32, device=dev).reshape(a.batch, nblk)
    lens = torch.full((a.batch,), seq, dtype=torch.int32, device=dev)
    q = torch.randn((a.batch, a.hq, 128), device=dev).to(torch.bfloat16)
    out = torch.empty_like(q)
    ws = ops.workspace(a.batch, a.hq, a.hkv, seq, dev)
    for p in pools:
        ops.decode_attention(q, p, bt, lens, out=out, max_seq_len=seq, ws=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for i in range(a.iters):
            ops.decode_attention(q, pools[i % layers], bt, lens, out=out, max_seq_len=seq, ws=ws)
    g.replay()
    torch.cuda.synchronize()
    times = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1) / a.iters)
    us = statistics.median(times) * 1e3
    alg = a.batch * seq * a.hkv * 512 + 2 * q.numel() * 2
    print(json.dumps({"batch": a.batch, "hq": a.hq, "hkv": a.hkv, "seq": seq, "variant": a.variant,
                      "us": us, "GBps": alg / us / 1e3, "alg_bytes": alg}), flush=True)
    del pools, g
    torch.cuda.empty_cache()
