"""How much would CUDA-graph replay of a whole decode step buy?  Times the
all-resident 8B step (cfg2r shape) and the 70B TP8 shard step (cfg4 shape,
K6 per layer), stream-launched vs replayed from one captured graph.  Replays
repeat the same positions (timing only, not a serving loop)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_10729_b200.core import PlacementMatrix, RequestState  # noqa: E402
from paper_2601_10729_b200.executor import B200Executor, ModelShape  # noqa: E402
from paper_2601_10729_b200.tp import HeadShard, TensorParallelDecoder  # noqa: E402


def probe(name, shape, B, prompt, hidden=None, shard=None, steps=10):
    dev = torch.device("cuda:0")
    cap = -(-(prompt + 64 + 1) // 16)
    batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=prompt, target_output_tokens=64)
             for i in range(B)]
    pm = PlacementMatrix.from_strides(range(B), shape.num_layers, [None] * B)
    ex = B200Executor(shape, device=dev, device_blocks=B * shape.num_layers * cap + 16,
                      host_blocks=16, fill="zeros", prefetch_next=False)
    ex.install(batch, pm)
    inp = ex.synthetic_inputs(B, step=0)
    tpd = TensorParallelDecoder(ex, shard, hidden, max_batch=B) if shard else None
    keep = []

    def run():
        # the executor's step without its host-side bookkeeping events (not capturable)
        desc, k = ex.prepare_step(batch, inp)
        keep.append(k)
        del keep[:-8]
        stream = torch.cuda.current_stream()
        if tpd is None:
            ex.runtime.decode_step(desc, stream)
            return
        out = k[1]
        hid = torch.empty((shape.num_layers, B, hidden), dtype=torch.bfloat16, device=dev)
        keep.append(hid)
        ex.runtime.step_begin(desc, stream)
        for l in range(shape.num_layers):
            ex.runtime.step_layers(1)
            tpd.proj(out, l, out=hid[l], stream=stream)
        ex.runtime.step_end()
    for _ in range(3):
        run()
    ex.drain()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        run()
    e1.record()
    ex.drain()
    torch.cuda.synchronize()
    stream_ms = e0.elapsed_time(e1) / steps
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        run()
    ex._inflight.clear()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    graph_ms = e0.elapsed_time(e1) / steps
    print(json.dumps({"step": name, "stream_ms": stream_ms, "graph_ms": graph_ms,
                      "gain": stream_ms / graph_ms - 1}), flush=True)
    del g
    if tpd:
        tpd.close()
    ex.close()


probe("8B all-resident B=16 32K", ModelShape(32, 32, 8), 16, 32760)
probe("70B TP8 shard B=32 64K", ModelShape(80, 8, 1), 32, 65528, hidden=8192, shard=HeadShard(0, 8, 64, 8))
