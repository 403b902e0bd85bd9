"""Per-CTA timeline of one stream-K K1 launch (globaltimer stamps, ofb_k1_trace).

Prints where the fixed cost of a launch goes: launch skew across CTAs, ramp
(entry -> first tile ready), streaming time distribution, end skew (last tile
of the earliest vs latest CTA) and the combine/exit tail.

    python tools/k1_trace.py --batch 32 --hq 8 --hkv 1 --seq 65536
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_10729_b200 import _native, ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--hq", type=int, default=8)
ap.add_argument("--hkv", type=int, default=1)
ap.add_argument("--seq", type=int, default=65536)
ap.add_argument("--dump", action="store_true")
a = ap.parse_args()

dev = torch.device("cuda:0")
ops.set_attention_kernel("stream")
lib = _native.load()
nblk = (a.seq + 15) // 16
pools = [torch.empty((a.batch * nblk, a.hkv, 2, 16, 128), dtype=torch.bfloat16, device=dev).normal_()
         for _ in range(3)]
bt = torch.arange(a.batch * nblk, dtype=torch.int32, device=dev).reshape(a.batch, nblk)
lens = torch.full((a.batch,), a.seq, dtype=torch.int32, device=dev)
q = torch.randn((a.batch, a.hq, 128), device=dev).to(torch.bfloat16)
out = torch.empty_like(q)
ws = ops.workspace(a.batch, a.hq, a.hkv, a.seq, dev)
trace = torch.zeros((448, 6), dtype=torch.int64, device=dev)
for i in range(4):   # back-to-back like a step; trace the last
    if i == 3:
        torch.cuda.synchronize()
        trace.zero_()
        lib.ofb_k1_trace(trace.data_ptr())
    ops.decode_attention(q, pools[i % 3], bt, lens, out=out, max_seq_len=a.seq, ws=ws)
torch.cuda.synchronize()
lib.ofb_k1_trace(None)
t = trace.cpu().numpy()
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = (t[:, :5] - t0) / 1e3   # us
entry, pdl, first, last, exit_ = rel.T
stream = last - first
res = {
    "ctas": int(len(t)), "kernel_span_us": float(exit_.max()),
    "entry_skew_us": [float(entry.min()), float(np.median(entry)), float(entry.max())],
    "pdl_wait_us_median": float(np.median(pdl - entry)),
    "ramp_us (entry->first tile)": [float((first - entry).min()), float(np.median(first - entry)), float((first - entry).max())],
    "streaming_us": [float(stream.min()), float(np.median(stream)), float(stream.max())],
    "last_tile_us": [float(last.min()), float(np.median(last)), float(last.max())],
    "tail_us (last tile -> exit)": [float((exit_ - last).min()), float(np.median(exit_ - last)), float((exit_ - last).max())],
    "exit_us": [float(exit_.min()), float(np.median(exit_)), float(exit_.max())],
    "alg_bytes": a.batch * a.seq * a.hkv * 512,
}
res["GBps_over_span"] = res["alg_bytes"] / res["kernel_span_us"] / 1e3
# per-CTA streaming rate vs its SM (which die / position)
per_cta = (res["alg_bytes"] / len(t)) / (stream * 1e3)
res["per_cta_GBps"] = [float(per_cta.min()), float(np.median(per_cta)), float(per_cta.max())]
slow = np.argsort(-last)[:8]
res["slowest_ctas"] = [{"cta": int(i), "sm": int(t[i, 5]), "last_tile_us": float(last[i]),
                        "first_us": float(first[i])} for i in slow]
# per SM: are the two co-resident CTAs slow together (SM-level) or split unevenly?
sm = t[:, 5]
by_sm = {}
for i in range(len(t)):
    by_sm.setdefault(int(sm[i]), []).append(i)
sm_rate = []
pair_ratio = []
for k, idx in by_sm.items():
    r = per_cta[idx]
    sm_rate.append(r.sum())
    if len(idx) == 2:
        pair_ratio.append(max(r) / min(r))
sm_rate = np.array(sm_rate)
res["sms"] = len(by_sm)
res["ctas_per_sm"] = sorted({len(v) for v in by_sm.values()})
res["per_sm_GBps"] = [float(sm_rate.min()), float(np.median(sm_rate)), float(sm_rate.max())]
res["intra_sm_rate_ratio"] = [float(min(pair_ratio)), float(np.median(pair_ratio)), float(max(pair_ratio))] if pair_ratio else None
if "--dump" in sys.argv:
    res["per_cta"] = [[int(sm[i]), float(per_cta[i]), float(first[i]), float(last[i]), float(exit_[i])]
                      for i in range(len(t))]
print(json.dumps(res, indent=1))
