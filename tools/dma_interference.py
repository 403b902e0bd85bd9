"""K1 alone vs K1 while 1 or 16 streams copy pinned host -> HBM."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2601_10729_b200 import _native, ops

dev = torch.device("cuda:0")
B, HKV, HQ, T = 16, 8, 32, 32768
nblk = (T + 15) // 16
pool = torch.randn((B * nblk, HKV, 2, 16, 128), device=dev).to(torch.bfloat16)
bt = torch.stack([torch.arange(nblk, dtype=torch.int32, device=dev) + r * nblk for r in range(B)])
lens = torch.full((B,), T, dtype=torch.int32, device=dev)
q = torch.randn((B, HQ, 128), device=dev).to(torch.bfloat16)
out = torch.empty_like(q)
ws = ops.workspace(B, HQ, HKV, T, dev)
lib = _native.load()
NB = 8 << 30
host = lib.ofb_host_alloc(NB)
dst = torch.empty(NB, dtype=torch.uint8, device=dev)
hbuf = torch.from_numpy(np.ctypeslib.as_array((__import__("ctypes").c_uint8 * 1).from_address(host))) if False else None

def k1_times(n=30):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(n + 2)]
    evs[0].record()
    for i in range(1, n + 2):
        ops.decode_attention(q, pool, bt, lens, max_seq_len=T, out=out, ws=ws)
        evs[i].record()
    evs[-1].synchronize()
    return float(np.median([evs[i].elapsed_time(evs[i + 1]) for i in range(1, n + 1)]))

res = {"alone": k1_times()}
import ctypes
cudart = ctypes.CDLL("libcudart.so.12")
for nstreams in (1, 4, 16):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    chunk = NB // nstreams
    for i, s in enumerate(streams):
        cudart.cudaMemcpyAsync(ctypes.c_void_p(dst.data_ptr() + i * chunk), ctypes.c_void_p(host + i * chunk),
                               ctypes.c_size_t(chunk), 1, ctypes.c_void_p(s.cuda_stream))
    res[f"with_{nstreams}_h2d_streams"] = k1_times()
    torch.cuda.synchronize()
print(json.dumps({k: round(v, 4) for k, v in res.items()}))
lib.ofb_host_free(host)
