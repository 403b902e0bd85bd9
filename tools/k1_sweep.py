"""K1 across batch / context / head layouts: graph-replayed back-to-back launches
(device time per launch), achieved GB/s against the measured copy peak, and the
variant the auto policy picks.  Prints one JSON line per point and a markdown
table at the end.

    python tools/k1_sweep.py > k1_sweep.md
"""
import json
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
rows = []
for hq, hkv, label in [(32, 8, "8B (32q/8kv)"), (8, 1, "70B TP8 shard (8q/1kv)"), (64, 8, "70B (64q/8kv)")]:
    for batch in (1, 4, 16, 32):
        for seq in (4096, 16384, 65536):
            nblk = (seq + 15) // 16
            layer_bytes = batch * nblk * hkv * 8192
            if layer_bytes > (6 << 30):
                continue
            layers = max(2, min(8, (1 << 30) // layer_bytes + 1))
            pools = [torch.empty((batch * nblk, hkv, 2, 16, 128), dtype=torch.bfloat16, device=dev).normal_()
                     for _ in range(layers)]
            bt = torch.arange(batch * nblk, dtype=torch.int32, device=dev).reshape(batch, nblk)
            lens = torch.full((batch,), seq, dtype=torch.int32, device=dev)
            q = torch.randn((batch, hq, 128), device=dev).to(torch.bfloat16)
            out = torch.empty_like(q)
            ws = ops.workspace(batch, hq, hkv, seq, dev)
            for p in pools:
                ops.decode_attention(q, p, bt, lens, out=out, max_seq_len=seq, ws=ws)
            iters = 16
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
            us = statistics.median(times) * 1e3
            alg = batch * seq * hkv * 512 + 2 * batch * hq * 128 * 2
            variant = {0: "stream-K", 1: "split", 3: "cluster", 4: "split2"}.get(int(lib.ofb_attention_variant_for(batch, hkv, seq)), "?")
            row = {"heads": label, "batch": batch, "seq": seq, "us": us, "GBps": alg / us / 1e3,
                   "frac_of_copy_peak": alg / us / 1e3 / PEAK, "variant": variant}
            rows.append(row)
            print(json.dumps(row), file=sys.stderr, flush=True)
            del pools, g
            torch.cuda.empty_cache()
print(f"| heads | B | context | variant | us | GB/s | / {PEAK:.0f} GB/s copy peak |")
print("|---|---|---|---|---|---|---|")
for r in rows:
    print(f"| {r['heads']} | {r['batch']} | {r['seq']} | {r['variant']} | {r['us']:.1f} | "
          f"{r['GBps']:.0f} | {r['frac_of_copy_peak']:.2f} |")
