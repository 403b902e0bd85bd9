"""The whole-decoder TP step (cfg4), the engine-driven TP executor, the
live-wall clock and step abort.

* ``TensorParallelLlama``: every layer's attention vs the CPU oracle (q from the
  QKV projection, KV from the slabs), the per-layer K3 append bit-exact against
  the projected k/v, and the whole hidden-state chain vs an fp32 torch
  restatement of the decoder layer (the attention output fed in from the GPU,
  itself checked against the oracle).
* ``TensorParallelExecutor`` under ``engine.Simulation``: parity-mode decisions
  equal the executor-less model run (src/engine.py:706-734).
* live-wall: a slow solve shifts the engine clock and the deliveries
  (src/engine.py:82-123, :612-632).
* a caller-side failure inside a split step propagates unchanged and leaves the
  runtime usable (``ofb_runtime_step_abort``).
"""

import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from paper_2601_10729_b200 import workload
from paper_2601_10729_b200.core import PlacementMatrix, RequestState, SloConfig, SystemProfile
from paper_2601_10729_b200.engine import RunConfig, Simulation
from paper_2601_10729_b200.policies import PolicyKind, make_policy

from test_executor_gpu import _check_step_outputs

pytestmark = pytest.mark.gpu


def _decoder(c1, L=3, hq=8, hkv=2, hidden=256, inter=512, B=3, seed=0, dev_extra=0):
    from paper_2601_10729_b200.executor import B200Executor, ModelShape
    from paper_2601_10729_b200.tp import HeadShard, TensorParallelLlama

    shape = ModelShape(L, hq, hkv)
    ex = B200Executor(shape, device_blocks=L * B * 40 + 2 * B * 40 + 64 + dev_extra,
                      host_blocks=L * B * 40 + 64, staging_slots=2, record_timing=True, seed=seed)
    dec = TensorParallelLlama(ex, HeadShard(0, 1, hq, hkv), hidden, inter, c1=c1, seed=seed,
                              max_batch=B)
    return ex, dec


def _batch(B=3):
    return [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=150 + 61 * i,
                         target_output_tokens=20) for i in range(B)]


def _rms(x, eps=1e-5):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps)


def _reference_chain(dec, ex, x_in):
    """fp32 decoder chain with the GPU attention output of every layer fed in."""
    L, B = ex.shape.num_layers, x_in.shape[0]
    x = x_in.float()
    qkv = []
    for l in range(L):
        w = {k: v.float() for k, v in dec.layer_weights(l).items()}
        a = _rms(x)
        qkv.append((a @ w["q"].t(), a @ w["k"].t(), a @ w["v"].t()))
        att = ex.last_output[l].float().reshape(B, -1)
        x = x + att @ w["o"].t()
        a = _rms(x)
        x = x + (F.silu(a @ w["gate"].t()) * (a @ w["up"].t())) @ w["down"].t()
    return x, qkv


@pytest.mark.parametrize("c1", ["k6", "nccl"])
def test_llama_decoder_step(c1):
    ex, dec = _decoder(c1)
    batch = _batch()
    L = ex.shape.num_layers
    rows = ((1, 0, 1), (0, 0, 0), (1, 1, 1))           # mixed resident / host-resident
    placement = PlacementMatrix(tuple(r.id for r in batch), L, rows)
    try:
        ex.install(batch, placement)
        g = torch.Generator(device=ex.device)
        g.manual_seed(5)
        for step in range(3):
            x_in = torch.randn((len(batch), dec.hidden), generator=g, device=ex.device).to(
                torch.bfloat16)
            out = dec.step(batch, x_in)
            torch.cuda.synchronize()
            ex.last_positions = np.array([r.total_tokens for r in batch], dtype=np.int32)
            _check_step_outputs(ex, batch)          # K1 vs oracle, q from the projection
            want, qkv = _reference_chain(dec, ex, x_in)
            q = ex.last_inputs["q"].float()
            kn, vn = ex.last_inputs["k_new"], ex.last_inputs["v_new"]
            for l in range(L):
                B = len(batch)
                torch.testing.assert_close(q[l].reshape(B, -1), qkv[l][0], rtol=3e-2, atol=3e-2)
                torch.testing.assert_close(kn[l].float().reshape(B, -1), qkv[l][1], rtol=3e-2,
                                           atol=3e-2)
                # K3 ran per layer: the token's slot holds the projected k / v bit for bit
                for b, r in enumerate(batch):
                    pos = r.total_tokens
                    bits = ex.slab_bits(r.id, l, pos // 16 + 1)
                    kb = kn[l, b].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
                    vb = vn[l, b].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
                    np.testing.assert_array_equal(bits[pos // 16, :, 0, pos % 16], kb)
                    np.testing.assert_array_equal(bits[pos // 16, :, 1, pos % 16], vb)
            torch.testing.assert_close(out.float(), want, rtol=5e-2, atol=5e-2)
            assert torch.isfinite(out.float()).all()
            for r in batch:
                r.record_generated_token()
    finally:
        dec.close()
        ex.close()


def test_c1_arms_agree():
    """K6 (fused projection) and the cuBLAS arm give the same decoder (world 1)."""
    outs = []
    for c1 in ("k6", "nccl"):
        ex, dec = _decoder(c1, seed=3)
        batch = _batch()
        placement = PlacementMatrix(tuple(r.id for r in batch), 3, ((1, 1, 1),) * 3)
        ex.install(batch, placement)
        x = torch.ones((3, dec.hidden), dtype=torch.bfloat16, device=ex.device)
        outs.append(dec.step(batch, x).float().clone())
        torch.cuda.synchronize()
        dec.close()
        ex.close()
    torch.testing.assert_close(outs[0], outs[1], rtol=3e-2, atol=3e-2)


def _toy_engine():
    prof = SystemProfile(num_layers=4, compute_base_ms=0.2, compute_per_token_ms=0.0004,
                         bandwidth_blocks_per_ms=12.0, gpu_block_budget=120, block_size=16,
                         prefill_per_token_ms=0.001)
    slo = SloConfig(tbt_target_ms=2.5, tpot_target_ms=2.5, window_min=2, window_max=6)
    trace = workload.Trace(tuple(workload.TraceRequest(i * 3, 90 + 37 * i, 6 + i % 3)
                                 for i in range(6)), {})
    return prof, slo, trace, RunConfig(max_batch=3)


def _strip(log):
    return [dict(r, payload={k: v for k, v in r["payload"].items()
                             if k not in ("measured_us", "wall_us")})
            if r["kind"] == "step" else r for r in log]


def test_tp_executor_under_engine():
    from paper_2601_10729_b200.executor import B200Executor, ModelShape
    from paper_2601_10729_b200.tp import HeadShard, TensorParallelExecutor, TensorParallelLlama

    prof, slo, trace, cfg = _toy_engine()

    def policy():
        return make_policy(PolicyKind.ORBIT, prof, slo, max_batch=3, token_cap=cfg.batch_token_cap)

    model = Simulation(trace, policy(), prof, slo, cfg).execute()
    ex = B200Executor.for_trace(trace, prof, shape=ModelShape(4, 8, 2), max_batch=3)
    dec = TensorParallelLlama(ex, HeadShard(0, 1, 8, 2), 256, 512, max_batch=3)
    tex = TensorParallelExecutor(dec)
    try:
        log = Simulation(trace, policy(), prof, slo, cfg, executor=tex).execute()
        assert _strip(log) == model
        steps = [r for r in log if r["kind"] == "step"]
        assert tex.steps == len(steps) and all(r["payload"]["measured_us"] > 0 for r in steps)
        assert not ex.slabs                       # every finished request was released
        wall = Simulation(trace, policy(), prof, slo, cfg, executor=tex, mode="live-wall").execute()
        wsteps = [r for r in wall if r["kind"] == "step"]
        assert all(r["payload"]["wall_us"] >= r["payload"]["measured_us"] for r in wsteps)
        assert sum(r["kind"] == "finish" for r in wall) == len(trace.requests)
    finally:
        tex.close()


def test_live_wall_slow_solve_shifts_deliveries(monkeypatch):
    """A solve that takes 40 ms of host time delays the next step by as much on the
    live-wall clock (and not on the live-device clock)."""
    from paper_2601_10729_b200 import engine
    from paper_2601_10729_b200.executor import B200Executor, ModelShape

    prof, slo, trace, cfg = _toy_engine()

    def run(mode):
        ex = B200Executor.for_trace(trace, prof, shape=ModelShape(4, 8, 2), max_batch=3)
        policy = make_policy(PolicyKind.ORBIT, prof, slo, max_batch=3, token_cap=cfg.batch_token_cap)
        log = Simulation(trace, policy, prof, slo, cfg, executor=ex, mode=mode).execute()
        ex.close()
        return log

    fast = run("live-wall")
    solves = [0]
    real_solve = engine._ref.solve

    def slow_solve(*a, **kw):
        import time

        solves[0] += 1
        time.sleep(0.04)
        return real_solve(*a, **kw)

    monkeypatch.setattr(engine._ref, "solve", slow_solve)
    slow = run("live-wall")
    device = run("live")
    assert solves[0] > 0

    def last_delivery(log):
        return max(r["time_us"] for r in log if r["kind"] == "deliver")

    def replan_steps(log):
        out, pending = [], False
        for r in log:
            if r["kind"] == "replan":
                pending = True
            elif r["kind"] == "step":
                if pending:
                    out.append(r["payload"]["wall_us"])
                pending = False
        return out

    # every step that followed a solve carries its 40 ms on the wall clock
    assert min(replan_steps(slow)) >= 40_000
    assert last_delivery(slow) - last_delivery(fast) >= 0.5 * 40_000 * len(replan_steps(slow))
    # the device clock does not see host time
    assert max(r["payload"]["measured_us"] for r in device if r["kind"] == "step") < 40_000


def test_step_abort_keeps_runtime_usable():
    from paper_2601_10729_b200.executor import B200Executor, ModelShape
    from paper_2601_10729_b200.tp import HeadShard, TensorParallelDecoder

    shape = ModelShape(3, 8, 2)
    batch = _batch()
    ex = B200Executor(shape, device_blocks=3 * 3 * 40 + 6 * 40 + 64, host_blocks=3 * 3 * 40 + 64,
                      staging_slots=2, record_timing=True)
    placement = PlacementMatrix(tuple(r.id for r in batch), 3, ((1, 0, 1), (0, 0, 0), (1, 1, 1)))
    tpd = TensorParallelDecoder(ex, HeadShard(0, 1, 8, 2), hidden=256, max_batch=3)
    try:
        ex.install(batch, placement)
        real = tpd.proj

        class Boom(RuntimeError):
            pass

        calls = [0]

        def failing(*a, **kw):
            calls[0] += 1
            if calls[0] == 2:
                raise Boom("projection failed")
            return real(*a, **kw)

        tpd.proj = failing
        with pytest.raises(Boom):
            tpd.step(batch, ex.synthetic_inputs(3, step=0))
        tpd.proj = real
        ex.drain()
        tpd.step(batch, ex.synthetic_inputs(3, step=1))
        torch.cuda.synchronize()
        ex.last_positions = np.array([r.total_tokens for r in batch], dtype=np.int32)
        _check_step_outputs(ex, batch)
    finally:
        tpd.close()
        ex.close()


@pytest.mark.parametrize("rows,hidden", [(32, 8192), (3, 4096), (1, 1024), (5, 16384)])
def test_rmsnorm_and_silu_mul_glue_match_fp32(rows, hidden):
    """The decoder glue kernels (ofb_rmsnorm, ofb_silu_mul) vs fp32 torch."""
    from paper_2601_10729_b200 import _native

    lib = _native.load()
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(rows + hidden)
    x = torch.randn((rows, hidden), generator=g, device=dev).to(torch.bfloat16)
    w = (1 + 0.1 * torch.randn((hidden,), generator=g, device=dev)).to(torch.bfloat16)
    out = torch.empty_like(x)
    s = torch.cuda.current_stream().cuda_stream
    _native.check(lib.ofb_rmsnorm(x.data_ptr(), w.data_ptr(), out.data_ptr(), rows, hidden, 1e-5, s),
                  "ofb_rmsnorm")
    want = _rms(x.float()) * w.float()
    torch.testing.assert_close(out.float(), want, rtol=2e-2, atol=1e-2)
    inter = hidden // 2
    gu = torch.randn((rows, 2 * inter), generator=g, device=dev).to(torch.bfloat16)
    act = torch.empty((rows, inter), dtype=torch.bfloat16, device=dev)
    _native.check(lib.ofb_silu_mul(gu.data_ptr(), act.data_ptr(), rows, inter, s), "ofb_silu_mul")
    want = F.silu(gu[:, :inter].float()) * gu[:, inter:].float()
    torch.testing.assert_close(act.float(), want, rtol=2e-2, atol=1e-2)


def _tp2_worker(rank, port, q):
    """One rank of a 2-way tensor-parallel whole-decoder step (gloo for the
    control plane; both processes share the box's GPU, so K6's exchange runs
    over CUDA IPC between the two contexts)."""
    import os

    import torch.distributed as dist

    from paper_2601_10729_b200.executor import B200Executor, ModelShape
    from paper_2601_10729_b200.tp import HeadShard, TensorParallelLlama

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        torch.cuda.set_device(0)
        L, B = 2, 3
        shard = HeadShard(rank, 2, 8, 2)
        ex = B200Executor(ModelShape(L, shard.local_q, shard.local_kv), device_blocks=L * B * 40 + 2 * B * 40 + 64,
                          host_blocks=L * B * 40 + 64, staging_slots=2, seed=11 + rank)
        dec = TensorParallelLlama(ex, shard, 256, 512, c1="k6", group=dist.group.WORLD, seed=0, max_batch=B)
        batch = _batch(B)
        rows = ((1, 0), (1, 1), (0, 1))               # host-resident slabs too (K2 + the runtime append)
        ex.install(batch, PlacementMatrix(tuple(r.id for r in batch), L, rows))
        g = torch.Generator(device=ex.device)
        g.manual_seed(99)                             # the same embeddings on both ranks
        res = []
        for _ in range(2):
            x_in = torch.randn((B, 256), generator=g, device=ex.device).to(torch.bfloat16)
            out = dec.step(batch, x_in)
            torch.cuda.synchronize()
            # numpy, not tensors: CPU tensors cross the queue by shared-memory handles
            # that die with this process
            npf = lambda t: t.float().cpu().numpy().copy()  # noqa: E731
            res.append({"x_in": npf(x_in), "out": out.view(torch.int16).cpu().numpy().copy(),
                        "attn": npf(ex.last_output), "q": npf(ex.last_inputs["q"]),
                        "w": [{k: npf(v) for k, v in dec.layer_weights(l).items()} for l in range(L)]})
            for r in batch:
                r.record_generated_token()
        dec.close()
        ex.close()
        q.put((rank, res))
    except Exception as exc:  # surfaced in the parent
        import traceback

        q.put((rank, f"error: {exc!r}\n{traceback.format_exc()}"))
    finally:
        dist.destroy_process_group()


def test_two_rank_whole_decoder_step_matches_the_unsharded_chain():
    """N = 2 KV-head shards of one decoder (two processes, one GPU): both ranks end
    every step with bit-identical hidden states, equal to an fp32 restatement of
    the UNSHARDED layer chain - q/k/v of each rank's heads, the o-projection and
    the MLP partials summed over the ranks by K6's exchange (with the residual add,
    the fused RMSNorms' row sums of squares and SwiGLU folded in)."""
    import multiprocessing as mp
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_tp2_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in (0, 1):
        assert not isinstance(res[r], str), res[r]
    def tensors(s):
        t = {k: torch.from_numpy(v) for k, v in s.items() if k != "w"}
        t["out"] = t["out"].view(torch.bfloat16)
        t["w"] = [{k: torch.from_numpy(v) for k, v in wl.items()} for wl in s["w"]]
        return t

    for step in range(2):
        s0, s1 = tensors(res[0][step]), tensors(res[1][step])
        assert torch.equal(s0["out"], s1["out"]), f"ranks disagree at step {step}"
        x = s0["x_in"]
        B = x.shape[0]
        for l in range(len(s0["w"])):
            a = _rms(x)
            for s in (s0, s1):        # each rank's q projection of its own heads
                torch.testing.assert_close(s["q"][l].reshape(B, -1), a @ s["w"][l]["q"].t(),
                                           rtol=3e-2, atol=3e-2)
            x = x + sum(s["attn"][l].reshape(B, -1) @ s["w"][l]["o"].t() for s in (s0, s1))
            a = _rms(x)
            x = x + sum((F.silu(a @ s["w"][l]["gate"].t()) * (a @ s["w"][l]["up"].t())) @ s["w"][l]["down"].t()
                        for s in (s0, s1))
        torch.testing.assert_close(s0["out"].float(), x, rtol=5e-2, atol=5e-2)


def _tp2_engine_worker(rank, port, q):
    """One rank of a 2-way TP deployment driven by the reference serving loop."""
    import os

    import torch.distributed as dist

    from paper_2601_10729_b200.executor import B200Executor, ModelShape
    from paper_2601_10729_b200.tp import HeadShard, TensorParallelExecutor, TensorParallelLlama

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        torch.cuda.set_device(0)
        prof, slo, trace, cfg = _toy_engine()
        shard = HeadShard(rank, 2, 8, 2)
        ex = B200Executor.for_trace(trace, prof, shape=ModelShape(4, shard.local_q, shard.local_kv), max_batch=3)
        dec = TensorParallelLlama(ex, shard, 256, 512, group=dist.group.WORLD, max_batch=3)
        tex = TensorParallelExecutor(dec, group=dist.group.WORLD)
        policy = make_policy(PolicyKind.ORBIT, prof, slo, max_batch=3, token_cap=cfg.batch_token_cap)
        log = Simulation(trace, policy, prof, slo, cfg, executor=tex).execute()
        steps = [r for r in log if r["kind"] == "step"]
        hidden = dec.last_hidden.view(torch.int16).cpu().numpy().copy()
        ok = bool(steps) and all(r["payload"]["measured_us"] > 0 for r in steps) and tex.steps == len(steps)
        tex.close()
        q.put((rank, (_strip(log), hidden, ok)))
    except Exception as exc:  # surfaced in the parent
        import traceback

        q.put((rank, f"error: {exc!r}\n{traceback.format_exc()}"))
    finally:
        dist.destroy_process_group()


def test_two_rank_tp_executor_under_engine():
    """Two ranks (two processes, one GPU) each run the reference serving loop over
    their KV-head shard: plans are recomputed per rank (C2, digest-checked), the
    measured step is the max over ranks, and both ranks' event logs equal the
    executor-less model run; the last hidden states are bit-identical."""
    import multiprocessing as mp
    import socket

    prof, slo, trace, cfg = _toy_engine()
    model = Simulation(trace, make_policy(PolicyKind.ORBIT, prof, slo, max_batch=3,
                                          token_cap=cfg.batch_token_cap), prof, slo, cfg).execute()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_tp2_engine_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in (0, 1):
        assert not isinstance(res[r], str), res[r]
        log, _hidden, ok = res[r]
        assert ok and log == model, f"rank {r}: decisions differ from the model run"
    assert (res[0][1] == res[1][1]).all(), "ranks' hidden states differ"
