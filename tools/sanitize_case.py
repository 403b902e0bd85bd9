"""Small K1/K3/K2/K4/K6 workload for compute-sanitizer (memcheck / racecheck / synccheck),
including steps that adopt the cross-step prefetch."""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import torch  # noqa: E402

from kvgen import make_case  # noqa: E402
from paper_2601_10729_b200 import ops  # noqa: E402
from paper_2601_10729_b200.core import PlacementMatrix, RequestState  # noqa: E402
from paper_2601_10729_b200.executor import B200Executor, ModelShape  # noqa: E402

dev = torch.device("cuda:0")
for variant in ("stream", "split", "split2", "cluster"):
    ops.set_attention_kernel(variant)
    for lens in ([700, 33, 1, 0, 255], [3000]):
        case = make_case(lens, 8, 2, seed=1)
        ops.decode_attention(case["q"].to(dev), case["pool"].to(dev),
                             torch.from_numpy(case["block_tables"]).to(dev),
                             torch.from_numpy(case["seq_lens"]).to(dev), scale=1 / math.sqrt(128))
# split combine with 5 / 2 / 1 thread groups dealing the splits (groups 1 / 2 / 16)
ops.set_attention_kernel("split")
for lens, hq, hkv in (([6000, 3], 2, 2), ([6001], 4, 2), ([8000, 70], 16, 1)):
    case = make_case(lens, hq, hkv, seed=2)
    ops.decode_attention(case["q"].to(dev), case["pool"].to(dev),
                         torch.from_numpy(case["block_tables"]).to(dev),
                         torch.from_numpy(case["seq_lens"]).to(dev), scale=1 / math.sqrt(128))
ops.set_attention_kernel("auto")

# planner GPU enumeration: histogram + windowed materialisation (tiny windows)
import os  # noqa: E402
import random  # noqa: E402

from paper_2601_10729_b200 import planner  # noqa: E402
from paper_2601_10729_b200.calibrate import b200_profile  # noqa: E402
from paper_2601_10729_b200 import defaults  # noqa: E402

os.environ["OFB_PLAN_WINDOW"] = "50"
rng = random.Random(3)
prof = b200_profile(8, 8, gpu_block_budget=400)
preqs = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=rng.randint(200, 900),
                      target_output_tokens=16) for i in range(4)]
planner.SOLVER = "native-gpu"
planner.solve_capacity_only(preqs, prof, defaults.default_slo(prof, 60.0), 1)
planner.SOLVER = "native"
del os.environ["OFB_PLAN_WINDOW"]

shape = ModelShape(4, 8, 2)
batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=200 + 70 * i, target_output_tokens=8)
         for i in range(3)]
ex = B200Executor(shape, device_blocks=300, host_blocks=300)
a = PlacementMatrix.from_strides([0, 1, 2], 4, [2, None, 1])
b = PlacementMatrix.from_strides([0, 1, 2], 4, [None, 1, 2])
ex.install(batch, a)
ex.decode_step(batch, a)
for r in batch:
    r.record_generated_token()
ex.install(batch, b)
for _ in range(3):           # same plan: steps 2 and 3 adopt the previous step's prefetch
    ex.decode_step(batch, b)
    for r in batch:
        r.record_generated_token()
assert ex.runtime.prefetch_stats()["adopted"] >= 2
torch.cuda.synchronize()
ex.close()

# K6 (tcgen05 o-projection; single rank: the exchange needs concurrently running
# peers, which the sanitizer's serialised launches cannot provide)
from paper_2601_10729_b200.collective import OprojAllReduce  # noqa: E402

for bsz, k, h in [(5, 128, 1024), (32, 1024, 2048)]:
    w = (torch.randn((2, h, k), device=dev) * k ** -0.5).to(torch.bfloat16)
    x = torch.randn((2, bsz, k), device=dev).to(torch.bfloat16)
    OprojAllReduce(w, bsz)(x, 1)
# K6 decoder-layer epilogues: fused RMSNorm (ss_out -> ss_in), SwiGLU, K3 fold
from paper_2601_10729_b200.collective import interleave_gate_up  # noqa: E402

bsz, k, h = 7, 256, 512
w = (torch.randn((2, h, k), device=dev) * k ** -0.5).to(torch.bfloat16)
x = torch.randn((bsz, h), device=dev).to(torch.bfloat16)
ss = torch.zeros((h // 128, 8), dtype=torch.float32, device=dev)
OprojAllReduce(w, 8)(torch.randn((2, bsz, k), device=dev).to(torch.bfloat16), 0, out=x, residual=x, ss_out=ss)
wgu = interleave_gate_up((torch.randn((2, 2 * 256, h), device=dev) * h ** -0.5).to(torch.bfloat16))
OprojAllReduce(wgu, 8)(x, 1, ss_in=ss, swiglu=True)
from paper_2601_10729_b200.tp import HeadShard, TensorParallelLlama  # noqa: E402

shape = ModelShape(2, 8, 2)
ex = B200Executor(shape, device_blocks=600, host_blocks=600, staging_slots=2)
dec = TensorParallelLlama(ex, HeadShard(0, 1, 8, 2), 256, 512, c1="k6", max_batch=3)
batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=150 + 61 * i, target_output_tokens=8)
         for i in range(3)]
pm = PlacementMatrix(tuple(r.id for r in batch), 2, ((1, 0), (1, 1), (0, 1)))
ex.install(batch, pm)
for _ in range(2):
    dec.step(batch, torch.randn((3, 256), device=dev).to(torch.bfloat16))
    for r in batch:
        r.record_generated_token()
torch.cuda.synchronize()
dec.close()
ex.close()

# attention-only all-resident steps: K1's consumers wait after the math (kv_ready 1),
# on the balanced narrow plan (8 KV heads, B=1, 4K: 17 splits x 8 pairs) and on the
# cost-model plan (1 KV head, B=2)
for (hq, hkv), B, ctx in (((32, 8), 1, 4096), ((8, 1), 2, 3000)):
    shape = ModelShape(3, hq, hkv)
    cap = -(-(ctx + 8) // 16)
    batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=ctx - 37 * i, target_output_tokens=8)
             for i in range(B)]
    ex = B200Executor(shape, device_blocks=B * 3 * cap + 16, host_blocks=16)
    ex.install(batch, PlacementMatrix.from_strides(range(B), 3, [None] * B))
    inp = ex.synthetic_inputs(B, step=0)
    for _ in range(3):
        ex.decode_step(batch, None, inp, sync=False)
    ex.drain()
    torch.cuda.synchronize()
    ex.close()
print("sanitize case done")
