"""Per-CTA timeline of the split K1 (globaltimer stamps, ofb_k1_trace_sized):
where a latency-bound launch spends its time.  Launches run back to back on
one stream (as inside a step, PDL on); the last one is traced.

Phases per CTA (medians, us from the earliest CTA entry):
  entry -> prologue (table + seq_lens loads, barrier init) -> first tile ready
  (first TMA round trip) -> ring drained (streaming + attention math) ->
  partial written (4-warp merge) -> ticket (fence + atomic) -> exit (the last
  CTA's combine).

    python tools/k1_split_trace.py --batch 1 --hq 8 --hkv 1 --seq 16384
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
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--hq", type=int, default=8)
ap.add_argument("--hkv", type=int, default=1)
ap.add_argument("--seq", type=int, default=16384)
ap.add_argument("--variant", default="split")
a = ap.parse_args()

dev = torch.device("cuda:0")
ops.set_attention_kernel(a.variant)
lib = _native.load()
nblk = (a.seq + 15) // 16
pools = [torch.empty((a.batch * nblk, a.hkv, 2, 16, 128), dtype=torch.bfloat16, device=dev).normal_()
         for _ in range(3)]
bt = torch.arange(a.batch * nblk, dtype=torch.int32, device=dev).reshape(a.batch, nblk)
lens = torch.full((a.batch,), a.seq, dtype=torch.int32, device=dev)
q = torch.randn((a.batch, a.hq, 128), device=dev).to(torch.bfloat16)
out = torch.empty_like(q)
ws = ops.workspace(a.batch, a.hq, a.hkv, a.seq, dev)
CAP = 4096
SLOTS = 8 if a.variant == "split" else 12
trace = torch.zeros((CAP, SLOTS), dtype=torch.int64, device=dev)
for i in range(6):
    if i == 5:
        torch.cuda.synchronize()
        trace.zero_()
        lib.ofb_k1_trace_sized(trace.data_ptr(), CAP)
        # the traced launch follows a busy predecessor, as in a step
        ops.decode_attention(q, pools[(i + 1) % 3], bt, lens, out=out, max_seq_len=a.seq, ws=ws)
    ops.decode_attention(q, pools[i % 3], bt, lens, out=out, max_seq_len=a.seq, ws=ws)
torch.cuda.synchronize()
lib.ofb_k1_trace_sized(None, CAP)
t = trace.cpu().numpy()
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
names = (["entry", "prologue", "first_tile", "drained", "partial", "ticket", "exit"] if a.variant == "split"
         else ["entry", "prologue", "first_tile", "drained", "merged", "cluster_sync", "gathered",
               "slice_written", "ticket", "exit"])
K = len(names)
rel = np.where(t[:, :K] > 0, (t[:, :K] - t0) / 1e3, np.nan)


def stats(x):
    x = x[~np.isnan(x)]
    if len(x) == 0:
        return None
    return [round(float(x.min()), 2), round(float(np.median(x)), 2), round(float(x.max()), 2)]


res = {"ctas": int(len(t)), "sms": int(len(set(t[:, SLOTS - 1].tolist()))),
       "span_us": round(float(np.nanmax(rel[:, K - 1])), 2)}
for i, n in enumerate(names):
    res[n + " (min/med/max us)"] = stats(rel[:, i])
for i in range(1, K):
    res[f"{names[i - 1]}->{names[i]} (min/med/max us)"] = stats(rel[:, i] - rel[:, i - 1])
res["alg_bytes"] = a.batch * a.seq * a.hkv * 512
res["GBps_over_span"] = res["alg_bytes"] / res["span_us"] / 1e3
print(json.dumps(res, indent=1))
