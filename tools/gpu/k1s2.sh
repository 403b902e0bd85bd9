# deferred-combine K1 (split2) vs default: parity on the kernel tests' shapes, in-step and standalone timing
python - <<'PY'
import math, torch, numpy as np, sys
sys.path.insert(0, ".")
import oracle
from paper_2601_10729_b200 import ops
dev = torch.device("cuda:0")
for (B, hq, hkv, seq) in [(1, 32, 8, 4096), (1, 8, 1, 16384), (3, 32, 8, 777), (2, 16, 2, 5000)]:
    nblk = (seq + 15) // 16
    pool = torch.randn((B * nblk + 4, hkv, 2, 16, 128), device=dev).to(torch.bfloat16)
    bt = torch.arange(B * nblk, dtype=torch.int32, device=dev).reshape(B, nblk)
    lens = torch.tensor([seq - 37 * b for b in range(B)], dtype=torch.int32, device=dev)
    q = torch.randn((B, hq, 128), device=dev).to(torch.bfloat16)
    outs = {}
    for v in ("split", "split2"):
        ops.set_attention_kernel(v)
        outs[v] = ops.decode_attention(q, pool, bt, lens, max_seq_len=seq).float()
    torch.cuda.synchronize()
    d = (outs["split"] - outs["split2"]).abs().max().item()
    print("split vs split2", B, hq, hkv, seq, "max|diff|", d)
ops.set_attention_kernel("auto")
PY
for v in split split2; do echo "== $v"; OFB_K1=$v timeout 300 python tools/small_step_probe.py | python -c "import sys,json
for l in sys.stdin:
  d=json.loads(l); print(d['shape'], d['B'], d['context'], round(d['us_per_layer'],2))"; done
OFB_K1=split2 timeout 600 python tools/k1_sweep.py 2>/dev/null | grep -E "\| 1 \||\| 4 \|" | head -20
