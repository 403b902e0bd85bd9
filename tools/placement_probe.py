"""How does the physical spacing of a layer's slabs in the pool affect K1?
One pool, 16 requests x E extents of 2053 blocks (64 KiB); layer 0 = extent 0 of
each request.  Times K1 back-to-back (events between launches)."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2601_10729_b200 import ops

dev = torch.device("cuda:0")
B, HKV, HQ, T = 16, 8, 32, 32768
nblk = (T + 15) // 16
cap = 2053
q = torch.randn((B, HQ, 128), device=dev).to(torch.bfloat16)
lens = torch.full((B,), T, dtype=torch.int32, device=dev)
out = torch.empty_like(q)
for variant in sys.argv[1:] or ["1", "2", "4", "8", "16", "32"]:
    E = int(variant.split(":")[0])
    gap = int(variant.split(":")[1]) if ":" in variant else 0
    blocks = B * E * (cap + gap)
    pool = torch.empty((blocks, HKV, 2, 16, 128), dtype=torch.bfloat16, device=dev)
    pool.view(torch.int16).random_(0, 16000)     # finite bf16 bit patterns
    tables = []
    for l in range(min(E, 4)):
        bt = torch.stack([torch.arange(nblk, dtype=torch.int32) + (r * E + l) * (cap + gap)
                          for r in range(B)]).to(dev)
        tables.append(bt)
    ws = ops.workspace(B, HQ, HKV, T, dev)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(18)]
    evs[0].record()
    for i in range(1, 18):
        ops.decode_attention(q, pool, tables[i % len(tables)], lens, max_seq_len=T, out=out, ws=ws)
        evs[i].record()
    evs[-1].synchronize()
    t = float(np.median([evs[i].elapsed_time(evs[i + 1]) for i in range(1, 17)]))
    gbs = B * T * HKV * 512 / (t * 1e-3) / 1e9
    print(json.dumps({"extents_per_request": E, "gap_blocks": gap, "ms": round(t, 4), "GBps": round(gbs)}), flush=True)
    del pool
    torch.cuda.empty_cache()
