"""Split-length sweep for the split K1 on latency-bound shapes: for each shape,
device time per launch (graph-replayed) at every OFB_K1_BPS value and at the
built-in plan, to fit the plan's cost model (stream time per block vs combine
time per split x query head).

    python tools/k1_bps_sweep.py > k1_bps.jsonl
"""
import argparse
import json
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_10729_b200 import ops  # noqa: E402

dev = torch.device("cuda:0")
ops.set_attention_kernel("split")
ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="1,8,1;4,8,1;16,8,1;1,32,8;4,32,8;1,64,8;1,16,1",
                help="batch,hq,hkv;...")
ap.add_argument("--seqs", default="4096,16384,65536")
ap.add_argument("--bps", default="2,4,8,12,16,24,32,48,64,96,128,256")
args = ap.parse_args()
SHAPES = [tuple(int(x) for x in t.split(",")) for t in args.shapes.split(";")]
SEQS = [int(x) for x in args.seqs.split(",")]
BPS = [None] + [int(x) for x in args.bps.split(",")]


def time_launch(q, pools, bt, lens, out, seq, ws, iters=20):
    layers = len(pools)
    for p in pools:
        ops.decode_attention(q, p, bt, lens, out=out, max_seq_len=seq, ws=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for i in range(iters):
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
        times.append(e0.elapsed_time(e1) / iters)
    del g
    return statistics.median(times) * 1e3


for batch, hq, hkv in SHAPES:
    for seq in SEQS:
        nblk = (seq + 15) // 16
        layer_bytes = batch * nblk * hkv * 8192
        layers = max(2, min(16, (1 << 30) // layer_bytes + 1))
        pools = [torch.empty((batch * nblk, hkv, 2, 16, 128), dtype=torch.bfloat16, device=dev).normal_()
                 for _ in range(layers)]
        bt = torch.arange(batch * nblk, dtype=torch.int32, device=dev).reshape(batch, nblk)
        lens = torch.full((batch,), seq, dtype=torch.int32, device=dev)
        q = torch.randn((batch, hq, 128), device=dev).to(torch.bfloat16)
        out = torch.empty_like(q)
        ws = ops.workspace(batch, hq, hkv, seq, dev)
        for bps in BPS:
            if bps is not None and (bps > nblk or -(-nblk // bps) > 256):
                continue
            if bps is None:
                os.environ.pop("OFB_K1_BPS", None)
            else:
                os.environ["OFB_K1_BPS"] = str(bps)
            us = time_launch(q, pools, bt, lens, out, seq, ws)
            print(json.dumps({"batch": batch, "hq": hq, "hkv": hkv, "seq": seq,
                              "bps": bps if bps is not None else "plan", "us": us}), flush=True)
        os.environ.pop("OFB_K1_BPS", None)
        del pools
        torch.cuda.empty_cache()
