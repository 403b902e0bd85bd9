"""K1 on the cfg2 executor's own resident layer vs a compact copy of the same data."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2601_10729_b200 import ops
from paper_2601_10729_b200.core import PlacementMatrix, RequestState
from paper_2601_10729_b200.executor import B200Executor, LLAMA31_8B

def timeit(fn, n=16):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(n + 2)]
    evs[0].record()
    for i in range(1, n + 2):
        fn(); evs[i].record()
    evs[-1].synchronize()
    return float(np.median([evs[i].elapsed_time(evs[i + 1]) for i in range(1, n + 1)]))

stride = [int(a) for a in sys.argv[1:2]] or [2]
B, L, cap = 16, 32, 2053
batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=32760, target_output_tokens=64) for i in range(B)]
pm = PlacementMatrix.from_strides(list(range(B)), L, [None if stride[0] == 0 else stride[0]] * B)
n_res = sum(r.count(1) for r in pm.rows)
ex = B200Executor(LLAMA31_8B, device_blocks=n_res * cap + 2 * B * cap + 16,
                  host_blocks=(L * B - n_res) * cap + 16, seed=0)
ex.install(batch, pm)
torch.cuda.synchronize()
layout = ex._layout(batch)
T = 32761
lens = torch.full((B,), T, dtype=torch.int32, device="cuda")
q = ex.synthetic_inputs(B, 0)["q"][0]
out = torch.empty_like(q)
ws = ex._workspace(B, T)
res = {}
for l in (0, 2):
    res[f"executor_layer{l}"] = timeit(lambda: ops.decode_attention(q, ex.pool.tensor, layout["tables"][l], lens, max_seq_len=T, out=out, ws=ws))
# compact copy of layer 0 into a fresh pool
nblk = (T + 15) // 16
tb = layout["tables"][0][:, :nblk].contiguous()
compact = torch.empty((B * nblk, 8, 2, 16, 128), dtype=torch.bfloat16, device="cuda")
for r in range(B):
    compact[r * nblk:(r + 1) * nblk] = ex.pool.tensor[tb[r].long()]
ctab = torch.stack([torch.arange(nblk, dtype=torch.int32, device="cuda") + r * nblk for r in range(B)])
res["compact_copy"] = timeit(lambda: ops.decode_attention(q, compact, ctab, lens, max_seq_len=T, out=out, ws=ws))
# same compact pool with probe-style random bits
compact2 = torch.empty_like(compact); compact2.view(torch.int16).random_(0, 16000)
res["compact_randbits"] = timeit(lambda: ops.decode_attention(q, compact2, ctab, lens, max_seq_len=T, out=out, ws=ws))
compact3 = torch.randn(compact.shape, device="cuda").to(torch.bfloat16)
res["compact_randn"] = timeit(lambda: ops.decode_attention(q, compact3, ctab, lens, max_seq_len=T, out=out, ws=ws))
q2 = torch.randn_like(q, dtype=torch.float32).to(torch.bfloat16)
res["compact_randn_q2"] = timeit(lambda: ops.decode_attention(q2, compact3, ctab, lens, max_seq_len=T, out=out, ws=ws))
print(json.dumps({k: round(v, 4) for k, v in res.items()}))
ex.close()
