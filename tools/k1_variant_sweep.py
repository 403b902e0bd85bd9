"""K1 work decompositions side by side on latency-bound and transitional shapes:
split (global last-CTA combine), split2 (a separate combine kernel) and cluster
(DSMEM combine) at cluster caps 16 / 8 / 4.  Graph-replayed back-to-back launches (device time per launch), and
each variant's output compared with the split kernel's (max |diff|).  One JSON
line per point on stderr, a markdown table on stdout.

    python tools/k1_variant_sweep.py [--quick] > k1_variants.md
"""
import json
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_10729_b200 import _native, ops  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent
try:
    PEAK = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
except Exception:
    PEAK = 6450.0

dev = torch.device("cuda:0")
lib = _native.load()
quick = "--quick" in sys.argv
VARIANTS = [("split", None), ("split2", None), ("cluster16", "16"), ("cluster8", "8"), ("cluster4", "4")]
shapes = []
for hq, hkv, label in [(32, 8, "8B"), (8, 1, "70B-TP8"), (64, 8, "70B")]:
    for batch in ((1, 4) if quick else (1, 2, 4, 8, 16)):
        for seq in ((4096, 16384) if quick else (1024, 4096, 16384, 65536)):
            if hkv * batch * seq > 8 * 16 * 16384:
                continue
            shapes.append((hq, hkv, label, batch, seq))


def timed(q, pools, bt, lens, out, seq, ws, iters=16):
    layers = len(pools)
    for p in pools:
        ops.decode_attention(q, p, bt, lens, out=out, max_seq_len=seq, ws=ws)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for i in range(iters):
            ops.decode_attention(q, pools[i % layers], bt, lens, out=out, max_seq_len=seq, ws=ws)
    g.replay()
    torch.cuda.synchronize()
    times = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1) / iters)
    return statistics.median(times) * 1e3


rows = []
for hq, hkv, label, batch, seq in shapes:
    nblk = (seq + 15) // 16
    layer_bytes = batch * nblk * hkv * 8192
    layers = max(2, min(8, (1 << 30) // layer_bytes + 1))
    pools = [torch.empty((batch * nblk, hkv, 2, 16, 128), dtype=torch.bfloat16, device=dev).normal_()
             for _ in range(layers)]
    perm = torch.randperm(batch * nblk, device=dev).to(torch.int32)
    bt = perm.reshape(batch, nblk).contiguous()
    lens = torch.full((batch,), seq, dtype=torch.int32, device=dev)
    lens[0] = seq - 5                                   # a partial last block
    q = torch.randn((batch, hq, 128), device=dev).to(torch.bfloat16)
    ws = ops.workspace(batch, hq, hkv, seq, dev)
    alg = (int(lens.sum()) * hkv * 512 + 2 * batch * hq * 128 * 2)
    row = {"heads": label, "batch": batch, "seq": seq}
    ref = None
    for name, cap in VARIANTS:
        if cap is None:
            os.environ.pop("OFB_K1_CLUSTER", None)
            ops.set_attention_kernel(name)
        else:
            os.environ["OFB_K1_CLUSTER"] = cap
            ops.set_attention_kernel("cluster")
        out = torch.empty_like(q)
        try:
            us = timed(q, pools, bt, lens, out, seq, ws)
        except Exception as exc:                        # noqa: BLE001
            row[name] = f"error: {exc}"[:120]
            continue
        ops.decode_attention(q, pools[0], bt, lens, out=out, max_seq_len=seq, ws=ws)
        torch.cuda.synchronize()
        if ref is None:
            ref = out.float().clone()
            diff = 0.0
        else:
            diff = float((out.float() - ref).abs().max())
        row[name] = round(us, 2)
        row[name + "_maxdiff"] = diff
    for name, cap in VARIANTS[2:]:
        os.environ["OFB_K1_CLUSTER"] = cap
        plan = ops.cluster_plan(batch, hkv, seq)
        row[name + "_plan"] = None if plan is None else (plan["cluster"], plan["clusters_per_pair"],
                                                          plan["blocks_per_cta"])
    os.environ.pop("OFB_K1_CLUSTER", None)
    ops.set_attention_kernel("auto")
    row["auto_pick"] = {0: "stream", 1: "split", 3: "cluster", 4: "split2"}.get(
        int(lib.ofb_attention_variant_for(batch, hkv, seq)), "?")
    row["alg_bytes"] = alg
    rows.append(row)
    print(json.dumps(row), file=sys.stderr, flush=True)
    del pools
    torch.cuda.empty_cache()

names = [n for n, _ in VARIANTS]
print(f"| heads | B | context | {' | '.join(n + ' us' for n in names)} | best | best GB/s | best / {PEAK:.0f} | "
      "cluster16 plan (C, P, blocks/CTA) |")
print("|---|---|---|" + "---|" * (len(names) + 4))
for r in rows:
    vals = {n: r[n] for n in names if isinstance(r.get(n), float)}
    best = min(vals, key=vals.get) if vals else "-"
    gbs = r["alg_bytes"] / vals[best] / 1e3 if vals else 0.0
    cells = " | ".join(f"{r[n]:.1f}" if isinstance(r.get(n), float) else "err" for n in names)
    print(f"| {r['heads']} | {r['batch']} | {r['seq']} | {cells} | {best} | {gbs:.0f} | {gbs / PEAK:.2f} | "
          f"{r.get('cluster16_plan')} |")
