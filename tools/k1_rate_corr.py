"""Are per-CTA (per-SM) K1 streaming rates stable across launches?  Six traced
launches on the same CTA->SM mapping: correlation of per-CTA and per-SM rates
(profiles/r01_summary.md: ~0.3, i.e. mostly transient contention)."""
import sys, json, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2601_10729_b200 import _native, ops
dev = torch.device("cuda:0"); ops.set_attention_kernel("stream"); lib = _native.load()
B, hq, hkv, seq = 32, 8, 1, 65536
nblk = (seq + 15) // 16
pools = [torch.empty((B * nblk, hkv, 2, 16, 128), dtype=torch.bfloat16, device=dev).normal_() for _ in range(3)]
bt = torch.arange(B * nblk, dtype=torch.int32, device=dev).reshape(B, nblk)
lens = torch.full((B,), seq, dtype=torch.int32, device=dev)
q = torch.randn((B, hq, 128), device=dev).to(torch.bfloat16); out = torch.empty_like(q)
ws = ops.workspace(B, hq, hkv, seq, dev)
traces = []
for rep in range(6):
    tr = torch.zeros((448, 6), dtype=torch.int64, device=dev)
    for i in range(3):
        if i == 2:
            torch.cuda.synchronize(); lib.ofb_k1_trace(tr.data_ptr())
        ops.decode_attention(q, pools[(i + rep) % 3], bt, lens, out=out, max_seq_len=seq, ws=ws)
    torch.cuda.synchronize(); lib.ofb_k1_trace(None)
    t = tr.cpu().numpy()[:296]
    rate = 1.0 / (t[:, 3] - t[:, 2])
    traces.append((t[:, 5].copy(), rate / rate.mean()))
sm0 = traces[0][0]
print("same SM per CTA across launches:", [float((tr[0] == sm0).mean()) for tr in traces])
r = np.array([tr[1] for tr in traces])
print("per-CTA rate corr between launches:", np.round(np.corrcoef(r)[0], 3).tolist())
# per-SM correlation
def per_sm(tr):
    d = {}
    for s, x in zip(*tr): d.setdefault(int(s), []).append(x)
    return np.array([np.mean(d[k]) for k in sorted(d)])
ps = np.array([per_sm(tr) for tr in traces])
print("per-SM rate corr:", np.round(np.corrcoef(ps)[0], 3).tolist())
print("spread per launch (max/min):", [round(float(x.max() / x.min()), 3) for x in r])
