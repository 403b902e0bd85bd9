"""``torch.ops.orbit``: the dispatcher registration of the data-path ops
 over the same C ABI as the ctypes binding.

CPU: the library loads, every op has its schema, the fake kernels propagate
metadata without a GPU, and a CPU tensor is refused (no CPU kernel exists).
GPU: a whole resident decode step (K3 append + K1 per layer) captured in a CUDA
graph through torch.ops and replayed equals the eager ctypes step bit for bit
and the CPU oracle within the north-star tolerance; the executor's step and
migrations through the torch binding equal the ctypes binding's bit for bit.
"""

import math

import numpy as np
import pytest
import torch

import oracle
from kvgen import bf16_bits, make_case

RTOL, ATOL = 2e-2, 1e-2

OPS = {
    "decode_attention": "orbit::decode_attention(Tensor q, Tensor kv_pool, Tensor block_tables, "
                        "Tensor seq_lens, int max_seq_len, float scale, Tensor ws) -> Tensor",
    "kv_append": "orbit::kv_append(Tensor k_new, Tensor v_new, Tensor(a!) kv_pool, "
                 "Tensor block_tables, Tensor positions, Tensor? host_slabs) -> ()",
    "kv_prefill": "orbit::kv_prefill(Tensor k, Tensor v, Tensor dst) -> ()",
    "decode_step": "orbit::decode_step(int runtime, int desc, Tensor(a!) out) -> ()",
    "migrate": "orbit::migrate(int runtime, Tensor dst, Tensor src, Tensor bytes, Tensor kinds, "
               "bool record_timing, Tensor stream_of) -> ()",
}


def _load():
    from paper_2601_10729_b200 import torch_ops

    torch_ops.load()
    return torch_ops


def test_library_registers_every_op():
    _load()
    for name, schema in OPS.items():
        assert str(getattr(torch.ops.orbit, name).default._schema) == schema
    assert "out" in torch.ops.orbit.decode_attention.overloads()


def test_fake_kernels_propagate_metadata():
    _load()
    from torch._subclasses.fake_tensor import FakeTensorMode

    with FakeTensorMode():
        q = torch.empty(4, 32, 128, dtype=torch.bfloat16)
        pool = torch.empty(64, 8, 2, 16, 128, dtype=torch.bfloat16)
        bt = torch.empty(4, 16, dtype=torch.int32)
        lens = torch.empty(4, dtype=torch.int32)
        ws = torch.empty(1 << 20, dtype=torch.uint8)
        out = torch.ops.orbit.decode_attention(q, pool, bt, lens, 256, 0.088, ws)
        assert out.shape == q.shape and out.dtype == torch.bfloat16


def test_cpu_tensors_are_refused():
    _load()
    case = make_case([40, 3], 8, 2, seed=1)
    with pytest.raises((NotImplementedError, RuntimeError)):
        torch.ops.orbit.decode_attention(case["q"], case["pool"],
                                         torch.from_numpy(case["block_tables"]),
                                         torch.from_numpy(case["seq_lens"]), 40, 0.088,
                                         torch.zeros(1 << 20, dtype=torch.uint8))


def _resident_step_inputs(L=3, hq=8, hkv=2, lens=(4000, 777, 33, 1), seed=11):
    g = torch.Generator().manual_seed(seed)
    B = len(lens)
    nblk = [(n + 1 + 15) // 16 for n in lens]          # room for the appended token
    width = max(nblk)
    total = L * sum(nblk) + 5
    pool = torch.randn((total, hkv, 2, 16, 128), generator=g).to(torch.bfloat16)
    perm = torch.randperm(total, generator=g).numpy().astype(np.int32)
    tables = np.full((L, B, width), -1, dtype=np.int32)
    cur = 0
    for l in range(L):
        for b, n in enumerate(nblk):
            tables[l, b, :n] = perm[cur:cur + n]
            cur += n
    q = torch.randn((L, B, hq, 128), generator=g).to(torch.bfloat16)
    k_new = torch.randn((L, B, hkv, 128), generator=g).to(torch.bfloat16)
    v_new = torch.randn((L, B, hkv, 128), generator=g).to(torch.bfloat16)
    pos = np.asarray(lens, dtype=np.int32)              # index of the appended token
    return dict(pool=pool, tables=tables, q=q, k_new=k_new, v_new=v_new, pos=pos)


@pytest.mark.gpu
def test_graph_captured_step_through_torch_ops_matches_eager_ctypes_and_oracle():
    torch_ops = _load()
    from paper_2601_10729_b200 import ops

    inp = _resident_step_inputs()
    dev = torch.device("cuda:0")
    L, B, hq = inp["q"].shape[:3]
    hkv = inp["pool"].shape[1]
    pos = torch.from_numpy(inp["pos"]).to(dev)
    lens = pos + 1
    max_len = int(inp["pos"].max()) + 1
    tables = torch.from_numpy(inp["tables"]).to(dev)
    q, kn, vn = (inp[k].to(dev) for k in ("q", "k_new", "v_new"))
    scale = 1.0 / math.sqrt(128)

    # eager, ctypes binding
    pool_a = inp["pool"].to(dev)
    ops.kv_append(kn, vn, pool_a, tables, pos)
    eager = torch.stack([ops.decode_attention(q[l], pool_a, tables[l], lens, max_seq_len=max_len,
                                              scale=scale) for l in range(L)])

    # captured, torch.ops binding
    pool_b = inp["pool"].to(dev)
    pristine = pool_b.clone()
    ws = torch.zeros(ops.workspace(B, hq, hkv, max_len, dev).numel(), dtype=torch.uint8, device=dev)
    out = torch.empty_like(q)

    def step():
        torch.ops.orbit.kv_append(kn, vn, pool_b, tables, pos, None)
        for l in range(L):
            torch.ops.orbit.decode_attention.out(q[l], pool_b, tables[l], lens, max_len, scale, ws,
                                                 out=out[l])

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()                                  # warm-up outside the capture
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    for _ in range(3):                          # replays: re-append is idempotent
        pool_b.copy_(pristine)
        out.zero_()
        graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(pool_b, pool_a)
    assert torch.equal(out, eager)

    host = bf16_bits(inp["pool"]).copy()
    for l in range(L):
        oracle.kv_append(bf16_bits(inp["k_new"][l]), bf16_bits(inp["v_new"][l]), host,
                         inp["tables"][l], inp["pos"])
    for l in range(L):
        want = oracle.decode_attention(bf16_bits(inp["q"][l]), host, inp["tables"][l],
                                       inp["pos"] + 1, scale)
        np.testing.assert_allclose(out[l].float().cpu().numpy(), want, rtol=RTOL, atol=ATOL)
    del torch_ops


@pytest.mark.gpu
def test_executor_step_and_migration_through_torch_binding_equal_ctypes():
    from paper_2601_10729_b200.core import PlacementMatrix, RequestState
    from paper_2601_10729_b200.executor import B200Executor, ModelShape

    shape = ModelShape(6, 8, 2)
    a = PlacementMatrix.from_strides([0, 1, 2], 6, [2, 3, None])
    b = PlacementMatrix.from_strides([0, 1, 2], 6, [3, None, 1])
    results = {}
    for binding in ("ctypes", "torch"):
        batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=300 + 50 * i,
                              target_output_tokens=40) for i in range(3)]
        ex = B200Executor(shape, device_blocks=6 * 3 * 30 + 64, host_blocks=6 * 3 * 30 + 64,
                          staging_slots=2, seed=5, binding=binding, record_timing=True)
        outs = []
        ex.install(batch, a)
        for step in range(4):
            if step == 2:
                ex.install(batch, b)        # K4 through orbit::migrate
            ex.decode_step(batch, b if step >= 2 else a)
            outs.append(ex.last_output.clone())
            for r in batch:
                r.record_generated_token()
        results[binding] = (torch.stack(outs).cpu(), dict(ex.migrated),
                            ex.last_timing["copy_bytes"])
        ex.close()
    assert torch.equal(results["ctypes"][0], results["torch"][0])
    assert results["ctypes"][1] == results["torch"][1] and results["torch"][1]["moves"] > 0
    assert results["ctypes"][2] == results["torch"][2]
