"""K6 microbenchmark: tcgen05 o-projection (world = 1) vs cuBLAS (torch.matmul),
and the fused all-reduce with N emulated ranks on one GPU.

Weights rotate over L layers (L x |W| > 126 MB L2), so every launch streams
its W_o rows from HBM.  Algorithmic bytes per launch = W (H x K x 2) + x
(B x K x 2) + out (B x H x 2).  CUDA events on the launching stream, median of
the per-launch intervals after warm-up.

    python tools/oproj_bench.py            -> one JSON line per shape
"""

import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2601_10729_b200.collective import OprojAllReduce, SymmetricBuffers  # noqa: E402

SHAPES = [  # name, B, K, H
    ("70B TP8", 32, 1024, 8192),
    ("70B TP4", 32, 2048, 8192),
    ("70B TP2", 32, 4096, 8192),
    ("70B TP1", 32, 8192, 8192),
    ("8B TP1 B16", 16, 4096, 4096),
    ("8B TP4 B16", 16, 1024, 4096),
    # the other projections of the 70B TP8 decoder step (same kernel, world 1)
    ("70B TP8 qkv", 32, 8192, 1280),
    ("70B TP8 gate_up", 32, 8192, 7168),
    ("70B TP8 down", 32, 3584, 8192),
]


def _time(fn, iters, layers, graph=True):
    """Median device time per call.  ``graph``: the calls are captured in a CUDA
    graph and replayed, so the number is kernel time, not Python launch cost."""
    for i in range(layers):       # warm-up over every layer (also configures the kernels)
        fn(i % layers)
    torch.cuda.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for i in range(iters):
                    fn(i % layers)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        times = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            b.synchronize()
            times.append(a.elapsed_time(b) / iters)
        return statistics.median(times)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(iters + 1)]
    evs[0].record()
    for i in range(iters):
        fn(i % layers)
        evs[i + 1].record()
    torch.cuda.synchronize()
    return statistics.median(evs[i].elapsed_time(evs[i + 1]) for i in range(iters))


def main():
    dev = torch.device("cuda:0")
    peak = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6450.0) \
        if (Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else 6450.0
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    for name, b, k, h in SHAPES:
        if only and name != only:
            continue
        # weights rotate past L2 unless --l2-resident (one layer: W stays in L2)
        layers = 1 if "--l2-resident" in sys.argv else max(4, (512 << 20) // (h * k * 2))
        w = (torch.randn((layers, h, k), device=dev) * k ** -0.5).to(torch.bfloat16)
        x = torch.randn((layers, b, k), device=dev).to(torch.bfloat16)
        op = OprojAllReduce(w, b)
        out = torch.empty((b, h), dtype=torch.bfloat16, device=dev)
        ms_k6 = _time(lambda l: op(x, l, out=out), 100, layers)
        wt = w.transpose(1, 2)   # [L, K, H] view: x @ W^T without a copy
        ms_cublas = _time(lambda l: torch.matmul(x[l], wt[l], out=out), 100, layers)
        ref = (x[0].float() @ w[0].float().T)
        err = (op(x, 0).float() - ref).abs().max().item()
        alg = h * k * 2 + b * k * 2 + b * h * 2
        line = {"shape": name, "B": b, "K": k, "H": h, "alg_bytes": alg,
                "k6_us": ms_k6 * 1e3, "k6_gbs": alg / (ms_k6 * 1e-3) / 1e9,
                "k6_frac": alg / (ms_k6 * 1e-3) / 1e9 / peak,
                "cublas_us": ms_cublas * 1e3, "cublas_gbs": alg / (ms_cublas * 1e-3) / 1e9,
                "speedup_vs_cublas": ms_cublas / ms_k6, "max_abs_err_vs_fp32": err}
        print(json.dumps(line), flush=True)
        del w, x, op
    # emulated ranks: the exchange path on one GPU (peer pointers are local, so
    # this times the kernel + protocol, not NVLink)
    for world, b, k, h in ([] if only or "--no-emulated" in sys.argv else [(2, 32, 1024, 8192)]):
        bufs = SymmetricBuffers.emulated(world, b, h, device=dev)
        layers = 8
        ops = [OprojAllReduce((torch.randn((layers, h, k), device=dev) * k ** -0.5).to(torch.bfloat16), b, bufs[r])
               for r in range(world)]
        xs = [torch.randn((layers, b, k), device=dev).to(torch.bfloat16) for _ in range(world)]
        streams = [torch.cuda.Stream(dev) for _ in range(world)]

        def step(l):
            for r in range(world):
                with torch.cuda.stream(streams[r]):
                    ops[r](xs[r], l)
            ev = torch.cuda.Event()
            for r in range(world):
                ev.record(streams[r])
                torch.cuda.current_stream().wait_event(ev)
        ms = _time(step, 50, layers, graph=False)
        for buf in bufs:
            buf.check()
        print(json.dumps({"emulated_world": world, "B": b, "K": k, "H": h,
                          "us_per_all_ranks_call": ms * 1e3,
                          "note": "all ranks share one GPU: not an NVLink number"}), flush=True)
        bufs[0].close()


if __name__ == "__main__":
    main()
