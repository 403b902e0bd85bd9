"""Per-CTA timeline of K6 launches (ofb_k6_trace): where the fixed cost goes.
Back-to-back launches over rotating W_o layers (like a step); the last traced."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_10729_b200 import _native  # noqa: E402
from paper_2601_10729_b200.collective import OprojAllReduce  # noqa: E402

b, k, h = [int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (32, 1024, 8192))]
dev = torch.device("cuda:0")
lib = _native.load()
layers = 8
w = (torch.randn((layers, h, k), device=dev) * k ** -0.5).to(torch.bfloat16)
x = torch.randn((layers, b, k), device=dev).to(torch.bfloat16)
op = OprojAllReduce(w, b)
tr = torch.zeros((512, 8), dtype=torch.int64, device=dev)
for i in range(6):
    if i == 5:
        torch.cuda.synchronize()
        lib.ofb_k6_trace(tr.data_ptr())
    op(x, i % layers)
torch.cuda.synchronize()
lib.ofb_k6_trace(None)
t = tr.cpu().numpy()
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = lambda c: (t[:, c][t[:, c] > 0] - t0) / 1e3  # noqa: E731
names = ["entry", "prologue_done", "acc_ready", "cluster_synced", "output_start", "exit", "rs_slice_store"]
res = {"ctas": int(len(t))}
for c, n in enumerate(names):
    v = rel(c)
    if len(v):
        res[n + "_us"] = [round(float(v.min()), 3), round(float(np.median(v)), 3), round(float(v.max()), 3)]
res["alg_MB"] = (h * k + b * k + b * h) * 2 / 1e6
print(json.dumps(res))
