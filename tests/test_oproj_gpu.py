"""K6 (C1): tcgen05 o-projection fused with the all-reduce over peer memory.

Checked against a plain PyTorch fp32 reference of the same op (the reference
kvsim has no multi-GPU path; the paper's decoder does
o_proj + NCCL all-reduce):
    hidden = sum_r x_r[layer] @ W_r[layer]^T
Tolerance: bf16 output (and bf16 partials on the wire) vs fp32 - 2e-2 rel /
3e-2 abs.  Every rank must hold bit-identical results (same values summed in
rank order).  Multi-rank runs use N ranks in one process on one GPU (the
kernel and the flag protocol are unchanged; peers are local pointers) and two
processes on one GPU exchanging CUDA IPC handles over gloo.
"""

import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu

RTOL, ATOL = 2e-2, 3e-2


def _inputs(world, layers, b, k, h, seed):
    g = torch.Generator().manual_seed(seed)
    xs = [torch.randn((layers, b, k), generator=g).to(torch.bfloat16) for _ in range(world)]
    ws = [(torch.randn((layers, h, k), generator=g) * (k * world) ** -0.5).to(torch.bfloat16)
          for _ in range(world)]
    return xs, ws


def _want(xs, ws, layer):
    return sum(x[layer].float() @ w[layer].float().T for x, w in zip(xs, ws))


@pytest.mark.parametrize("b,k,h", [
    (32, 1024, 8192),     # 70B TP8 shard: 8 q heads x 128 -> hidden 8192
    (32, 8192, 8192),     # 70B TP1
    (32, 8192, 1280),     # 70B TP8 q/k/v projection: 10 tiles x 8-CTA clusters
    (16, 1024, 4096),     # 8B TP4
    (5, 128, 1024),       # toy, ragged batch
    (256, 256, 1024),     # max batch
    (1, 64, 128),         # smallest geometry
])
def test_single_rank_projection_matches_fp32(b, k, h):
    from paper_2601_10729_b200.collective import OprojAllReduce

    dev = torch.device("cuda:0")
    xs, ws = _inputs(1, 3, b, k, h, seed=b + k + h)
    op = OprojAllReduce(ws[0].to(dev), max_batch=b)
    x = xs[0].to(dev)
    for layer in (0, 2):
        got = op(x, layer)
        torch.cuda.synchronize()
        torch.testing.assert_close(got.float().cpu(), _want(xs, ws, layer), rtol=RTOL, atol=ATOL)
        again = op(x, layer)
        torch.cuda.synchronize()
        assert torch.equal(got, again), "split-K reduction must be deterministic"


@pytest.mark.parametrize("world,b,k,h", [
    (2, 32, 1024, 8192),  # 70B TP8 shard geometry, two ranks
    (4, 16, 256, 1024),
    (8, 8, 128, 512),
])
def test_emulated_ranks_all_reduce(world, b, k, h):
    from paper_2601_10729_b200.collective import OprojAllReduce, SymmetricBuffers

    dev = torch.device("cuda:0")
    layers = 2
    bufs = SymmetricBuffers.emulated(world, b, h, device=dev)
    try:
        streams = [torch.cuda.Stream(dev) for _ in range(world)]
        for call in range(5):       # both inbox parities, reused; inputs change every call
            xs, ws = _inputs(world, layers, b, k, h, seed=100 * world + call)
            ops = [OprojAllReduce(ws[r].to(dev), b, bufs[r]) for r in range(world)]
            xd = [x.to(dev) for x in xs]
            torch.cuda.synchronize()
            outs = []
            for r in range(world):
                with torch.cuda.stream(streams[r]):
                    outs.append(ops[r](xd[r], call % layers))
            torch.cuda.synchronize()
            for buf in bufs:
                buf.check()
            want = _want(xs, ws, call % layers)
            for r in range(world):
                assert torch.equal(outs[r], outs[0]), f"rank {r} differs from rank 0 (call {call})"
            torch.testing.assert_close(outs[0].float().cpu(), want, rtol=RTOL, atol=ATOL)
    finally:
        bufs[0].close()


def test_missing_peer_times_out_and_is_reported():
    """A rank whose peer never launches must not hang the GPU: the tile wait is
    bounded, the status word is raised and check() turns it into an error."""
    from paper_2601_10729_b200.collective import OprojAllReduce, SymmetricBuffers

    dev = torch.device("cuda:0")
    b, k, h = 8, 128, 256
    bufs = SymmetricBuffers.emulated(2, b, h, device=dev)
    try:
        xs, ws = _inputs(2, 1, b, k, h, seed=5)
        op = OprojAllReduce(ws[0].to(dev), b, bufs[0], timeout_ns=20_000_000)
        op(xs[0].to(dev), 0)          # rank 1 never runs
        torch.cuda.synchronize()
        with pytest.raises(RuntimeError, match="never arrived"):
            bufs[0].check()
    finally:
        bufs[0].close()


def test_exchange_refuses_a_grid_the_gpu_cannot_hold_at_once():
    """Every tile's CTA spins on its peers' flags, so the exchange is only safe
    when the whole grid is co-resident: a launch with more tiles than the GPU
    co-schedules (here 200 hidden tiles of one CTA each, > 148 SMs at one
    200 KiB CTA per SM) is refused before anything runs, while the same shape
    without an exchange (world 1) still launches."""
    from paper_2601_10729_b200.collective import OprojAllReduce, SymmetricBuffers

    dev = torch.device("cuda:0")
    b, k, h = 8, 128, 128 * 200
    bufs = SymmetricBuffers.emulated(2, b, h, device=dev)
    try:
        xs, ws = _inputs(2, 1, b, k, h, seed=9)
        op = OprojAllReduce(ws[0].to(dev), b, bufs[0])
        with pytest.raises(RuntimeError, match="co-schedules"):
            op(xs[0].to(dev), 0)
        torch.cuda.synchronize()
        single = OprojAllReduce(ws[0].to(dev), b)
        out = single(xs[0].to(dev), 0)
        torch.cuda.synchronize()
        want = xs[0][0].float() @ ws[0][0].float().T
        torch.testing.assert_close(out.float().cpu(), want, rtol=RTOL, atol=ATOL)
    finally:
        bufs[0].close()


@pytest.mark.parametrize("splits", [1, 2, 3, 5, 8])
def test_cluster_split_counts_agree_with_fp32(monkeypatch, splits):
    """Every cluster size of the split-K reduction (3 and 5: non-power-of-two
    clusters, uneven K ranges) gives the fp32 result through the plain, the
    residual and the column-parts epilogues, and is deterministic."""
    from paper_2601_10729_b200.collective import OprojAllReduce

    dev = torch.device("cuda:0")
    b, k, h = 19, 4096, 1280          # 64 K chunks: >= 4 per CTA even at 8 splits
    xs, ws = _inputs(1, 2, b, k, h, seed=40 + splits)
    monkeypatch.setenv("OFB_K6_SPLITS", str(splits))
    op = OprojAllReduce(ws[0].to(dev), max_batch=32)
    x = xs[0].to(dev)
    want = xs[0][1].float() @ ws[0][1].float().T
    plain = op(x, 1)
    res = torch.randn((b, h), generator=torch.Generator().manual_seed(3)).to(torch.bfloat16)
    out = res.to(dev).clone()
    op(x, 1, out=out, residual=out)
    parts = [torch.empty((b, c), dtype=torch.bfloat16, device=dev) for c in (1024, 128, 128)]
    op(x, 1, parts=parts)
    again = op(x, 1)
    torch.cuda.synchronize()
    torch.testing.assert_close(plain.float().cpu(), want, rtol=RTOL, atol=ATOL)
    torch.testing.assert_close(out.float().cpu(), want + res.float(), rtol=RTOL, atol=ATOL)
    assert torch.equal(torch.cat(parts, 1), plain), "parts must equal the single output bit for bit"
    assert torch.equal(again, plain), "split-K reduction must be deterministic"


def _ipc_worker(rank, world, port, b, k, h, q):
    import torch.distributed as dist

    from paper_2601_10729_b200.collective import OprojAllReduce, SymmetricBuffers

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        xs, ws = _inputs(world, 2, b, k, h, seed=77)
        buf = SymmetricBuffers(world, rank, b, h, device="cuda:0")
        op = OprojAllReduce(ws[rank].cuda(), b, buf)
        x = xs[rank].cuda()
        outs = []
        for call in range(3):
            dist.barrier()
            outs.append(op(x, call % 2).cpu())
        buf.check()
        dist.barrier()
        buf.close()
        q.put((rank, [o.view(torch.int16).numpy().tobytes() for o in outs]))
    except Exception as exc:  # surfaced in the parent
        q.put((rank, f"error: {exc!r}"))
    finally:
        dist.destroy_process_group()


def test_two_processes_exchange_ipc_handles_on_one_gpu():
    import numpy as np
    import torch.multiprocessing as mp

    b, k, h, world = 16, 256, 1024, 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, b, k, h, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
    assert res[0] == res[1], "ranks disagree"
    xs, ws = _inputs(world, 2, b, k, h, seed=77)
    for call, raw in enumerate(res[0]):
        got = torch.from_numpy(np.frombuffer(raw, dtype=np.int16).copy()).view(torch.bfloat16).view(b, h)
        torch.testing.assert_close(got.float(), _want(xs, ws, call % 2), rtol=RTOL, atol=ATOL)


def test_column_parts_equal_the_single_output():
    """One K6 launch writing the q / k / v column ranges straight into three
    tensors gives exactly the columns of the single-output projection."""
    from paper_2601_10729_b200.collective import OprojAllReduce

    dev = torch.device("cuda:0")
    b, k, h = 5, 512, 128 * 10           # 8 q tiles + 1 k tile + 1 v tile
    xs, ws = _inputs(1, 2, b, k, h, seed=21)
    op = OprojAllReduce(ws[0].to(dev), b)
    x = xs[0].to(dev)
    whole = op(x, 1)
    qv = torch.empty((b, 1024), dtype=torch.bfloat16, device=dev)
    kv = torch.empty((b, 128), dtype=torch.bfloat16, device=dev)
    vv = torch.empty((b, 128), dtype=torch.bfloat16, device=dev)
    op(x, 1, parts=[qv, kv, vv])
    torch.cuda.synchronize()
    assert torch.equal(qv, whole[:, :1024])
    assert torch.equal(kv, whole[:, 1024:1152])
    assert torch.equal(vv, whole[:, 1152:])
    with pytest.raises(ValueError):
        op(x, 1, parts=[qv, kv])          # columns do not add up to hidden


def test_fused_residual_adds_before_the_rounding():
    from paper_2601_10729_b200.collective import OprojAllReduce

    dev = torch.device("cuda:0")
    b, k, h = 7, 256, 512
    xs, ws = _inputs(1, 1, b, k, h, seed=31)
    op = OprojAllReduce(ws[0].to(dev), b)
    resid = torch.randn((b, h), device=dev).to(torch.bfloat16)
    want = resid.float() + xs[0][0].to(dev).float() @ ws[0][0].to(dev).float().T
    x_res = resid.clone()
    op(xs[0].to(dev), 0, out=x_res, residual=x_res)       # in place: x += proj
    torch.cuda.synchronize()
    torch.testing.assert_close(x_res.float(), want, rtol=RTOL, atol=ATOL)


def _rms(x, eps=1e-5):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps)


def _tile_sumsq(y, max_batch):
    """fp32 [H/128, max_batch]: per 128-column tile, each row's sum of squares."""
    b, h = y.shape
    out = torch.zeros((h // 128, max_batch), dtype=torch.float32)
    out[:, :b] = y.float().pow(2).reshape(b, h // 128, 128).sum(-1).T
    return out


def test_fused_rmsnorm_ss_out_and_ss_in():
    """A producer K6 (residual add) leaves each tile's row sums of squares of its
    final output; a consumer K6 fed a 2-D x (one input for every layer) and that
    ss scales its rows by rsqrt(mean(x^2)+eps) - RMSNorm(x) . W^T; the first
    layer's ss comes from ofb_row_sumsq."""
    from paper_2601_10729_b200 import _native
    from paper_2601_10729_b200.collective import OprojAllReduce

    dev = torch.device("cuda:0")
    b, k, h, mb = 13, 512, 1024, 16
    xs, ws = _inputs(1, 2, b, k, h, seed=21)
    prod = OprojAllReduce(ws[0].to(dev), max_batch=mb)
    res = torch.randn((b, h), generator=torch.Generator().manual_seed(8)).to(torch.bfloat16)
    x = res.to(dev).clone()
    ss = torch.zeros((h // 128, mb), dtype=torch.float32, device=dev)
    prod(xs[0].to(dev), 1, out=x, residual=x, ss_out=ss)
    torch.cuda.synchronize()
    torch.testing.assert_close(ss.cpu(), _tile_sumsq(x.cpu(), mb), rtol=1e-5, atol=1e-4)
    # ofb_row_sumsq gives the same layout for an arbitrary x
    ss2 = torch.zeros_like(ss)
    _native.check(_native.load().ofb_row_sumsq(x.data_ptr(), ss2.data_ptr(), b, h, mb, None), "row_sumsq")
    torch.cuda.synchronize()
    torch.testing.assert_close(ss2.cpu(), ss.cpu(), rtol=1e-6, atol=1e-5)
    # consumer: 3 layers of W [512, h], one x for every layer
    w_c = (torch.randn((3, 512, h), generator=torch.Generator().manual_seed(9)) * h ** -0.5).to(torch.bfloat16)
    cons = OprojAllReduce(w_c.to(dev), max_batch=mb)
    for layer in (0, 2):
        got = cons(x, layer, ss_in=ss, eps=1e-5)
        torch.cuda.synchronize()
        want = _rms(x.float().cpu()) @ w_c[layer].float().T
        torch.testing.assert_close(got.float().cpu(), want, rtol=RTOL, atol=ATOL)


def test_swiglu_epilogue():
    """Gate/up rows interleaved per 64: the K6 epilogue emits silu(gate) * up of
    the rounded projections (with the fused RMSNorm row scale)."""
    import torch.nn.functional as F

    from paper_2601_10729_b200.collective import OprojAllReduce, deinterleave_gate_up, interleave_gate_up

    dev = torch.device("cuda:0")
    b, k, inter, mb = 9, 256, 384, 16
    g = torch.Generator().manual_seed(31)
    w_gu = (torch.randn((2, 2 * inter, k), generator=g) * k ** -0.5).to(torch.bfloat16)
    assert torch.equal(deinterleave_gate_up(interleave_gate_up(w_gu)), w_gu)
    op = OprojAllReduce(interleave_gate_up(w_gu).to(dev), max_batch=mb)
    x = torch.randn((b, k), generator=g).to(torch.bfloat16)
    ss = torch.zeros((k // 128, mb), dtype=torch.float32)
    ss[:, :b] = x.float().pow(2).reshape(b, k // 128, 128).sum(-1).T
    act = op(x.to(dev), 1, ss_in=ss.to(dev), eps=1e-5, swiglu=True)
    torch.cuda.synchronize()
    a = _rms(x.float())
    gu = (a @ w_gu[1].float().T).to(torch.bfloat16).float()
    want = F.silu(gu[:, :inter]) * gu[:, inter:]
    assert act.shape == (b, inter)
    torch.testing.assert_close(act.float().cpu(), want, rtol=RTOL, atol=ATOL)


def test_exchange_leaves_identical_row_sums_on_every_rank():
    """With the all-reduce (world 2, emulated), ss_out is computed from the
    reduced output in a fixed order: identical on both ranks and equal to the
    output's tile sums."""
    from paper_2601_10729_b200.collective import OprojAllReduce, SymmetricBuffers

    dev = torch.device("cuda:0")
    world, b, k, h = 2, 11, 256, 1024
    bufs = SymmetricBuffers.emulated(world, b, h, device=dev)
    try:
        xs, ws = _inputs(world, 1, b, k, h, seed=55)
        ops = [OprojAllReduce(ws[r].to(dev), b, bufs[r]) for r in range(world)]
        res = torch.randn((b, h), generator=torch.Generator().manual_seed(4)).to(torch.bfloat16).to(dev)
        outs = [res.clone() for _ in range(world)]
        sss = [torch.zeros((h // 128, b), dtype=torch.float32, device=dev) for _ in range(world)]
        streams = [torch.cuda.Stream(dev) for _ in range(world)]
        torch.cuda.synchronize()
        for r in range(world):
            with torch.cuda.stream(streams[r]):
                ops[r](xs[r].to(dev), 0, out=outs[r], residual=outs[r], ss_out=sss[r])
        torch.cuda.synchronize()
        for buf in bufs:
            buf.check()
        assert torch.equal(outs[0], outs[1]) and torch.equal(sss[0], sss[1])
        torch.testing.assert_close(sss[0].cpu(), _tile_sumsq(outs[0].cpu(), b), rtol=1e-5, atol=1e-4)
        want = _want(xs, ws, 0) + res.float().cpu()
        torch.testing.assert_close(outs[0].float().cpu(), want, rtol=RTOL, atol=ATOL)
    finally:
        bufs[0].close()
