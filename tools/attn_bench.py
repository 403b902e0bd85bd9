"""Micro-benchmark of K1 alone: one layer, KV resident in HBM, CUDA-event timed."""
import argparse, json, math, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2601_10729_b200 import ops

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--hq", type=int, default=32)
ap.add_argument("--hkv", type=int, default=8)
ap.add_argument("--seq", type=int, default=32768)
ap.add_argument("--layers", type=int, default=8, help="distinct layer pools rotated (defeats L2)")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--variant", default="auto", choices=["stream", "split", "auto"])
ap.add_argument("--pin-gib", type=int, default=0, help="allocate this much mapped pinned host memory first")
ap.add_argument("--pool-extra-gib", type=int, default=0, help="extra unused device pool memory")
a = ap.parse_args()
dev = torch.device("cuda:0")
ops.set_attention_kernel(a.variant)
from paper_2601_10729_b200 import _native
_pinned = _native.load().ofb_host_alloc(a.pin_gib << 30) if a.pin_gib else None
_extra = torch.empty(a.pool_extra_gib << 30, dtype=torch.uint8, device=dev) if a.pool_extra_gib else None
nblk = (a.seq + 15) // 16
pools = [torch.empty((a.batch * nblk, a.hkv, 2, 16, 128), dtype=torch.bfloat16, device=dev).normal_() for _ in range(a.layers)]
bt = torch.arange(a.batch * nblk, dtype=torch.int32, device=dev).reshape(a.batch, nblk)
lens = torch.full((a.batch,), a.seq, dtype=torch.int32, device=dev)
q = torch.randn((a.batch, a.hq, 128), device=dev).to(torch.bfloat16)
out = torch.empty_like(q)
ws = ops.workspace(a.batch, a.hq, a.hkv, a.seq, dev)
for p in pools:
    ops.decode_attention(q, p, bt, lens, out=out, max_seq_len=a.seq, ws=ws)
torch.cuda.synchronize()
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.iters)]
for i in range(a.iters):
    evs[i][0].record(); ops.decode_attention(q, pools[i % a.layers], bt, lens, out=out, max_seq_len=a.seq, ws=ws); evs[i][1].record()
torch.cuda.synchronize()
ms = sorted(s.elapsed_time(e) for s, e in evs)
bytes_ = a.batch * a.seq * a.hkv * 2 * 128 * 2 + 2 * q.numel() * 2
med = ms[len(ms) // 2]
print(json.dumps({"shape": vars(a), "median_ms": med, "best_ms": ms[0], "GBps_median": bytes_ / med / 1e6,
                  "GBps_best": bytes_ / ms[0] / 1e6, "device_info": ops.device_info()}))
