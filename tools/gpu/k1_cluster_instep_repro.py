import os, sys, ctypes, traceback
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_10729_b200 import _native
from paper_2601_10729_b200.core import PlacementMatrix, RequestState
from paper_2601_10729_b200.executor import B200Executor, ModelShape
lib = _native.load()
for B, ctx in [(1, 4096), (4, 4096), (1, 1024), (4, 1024)]:
    shape = ModelShape(32, 32, 8)
    cap = -(-(ctx + 64 + 1) // 16)
    batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=ctx, target_output_tokens=64) for i in range(B)]
    pm = PlacementMatrix.from_strides(range(B), 32, [None] * B)
    ex = B200Executor(shape, device_blocks=B * 32 * cap + 16, host_blocks=16, fill="zeros")
    ex.install(batch, pm)
    inp = ex.synthetic_inputs(B, step=0)
    C, P, bps, st = (ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32())
    try:
        ex.decode_step(batch, None, inp, sync=True)
        print(B, ctx, "ok", flush=True)
    except Exception as e:
        print(B, ctx, "FAIL", e, flush=True)
    ex.close()
