"""The B200 executor under the engine: bit-exact decisions, physical residency
equal to the BlockTable, every step's attention output vs the CPU oracle,
byte-exact K4 migrations (evict -> restore round trips) and K2 fetch volume
equal to the reference's blocks_to_fetch."""

import math

import numpy as np
import pytest
import torch

import oracle
from paper_2601_10729_b200 import defaults, workload
from paper_2601_10729_b200.core import PlacementMatrix, RequestState, SloConfig, SystemProfile
from paper_2601_10729_b200.engine import RunConfig, Simulation
from paper_2601_10729_b200.latency import blocks_to_fetch
from paper_2601_10729_b200.policies import PolicyKind, make_policy

pytestmark = pytest.mark.gpu

RTOL, ATOL = 2e-2, 1e-2


def _executor(shape, **kw):
    from paper_2601_10729_b200.executor import B200Executor
    return B200Executor(shape, **kw)


def _check_step_outputs(ex, batch):
    """Oracle attention for every (layer, request) of the last step."""
    L = ex.shape.num_layers
    pos = ex.last_positions
    scale = 1.0 / math.sqrt(128)
    q = ex.last_inputs["q"].float().cpu()
    out = ex.last_output.float().cpu().numpy()
    for l in range(L):
        blocks = [int(p) // 16 + 1 for p in pos]
        slabs = [ex.slab_bits(r.id, l, n) for r, n in zip(batch, blocks)]
        pool = np.concatenate(slabs, axis=0)
        width = max(blocks)
        bt = np.full((len(batch), width), -1, dtype=np.int32)
        cur = 0
        for b, n in enumerate(blocks):
            bt[b, :n] = np.arange(cur, cur + n)
            cur += n
        qb = q[l].to(torch.bfloat16).contiguous().view(torch.int16).numpy().view(np.uint16)
        want = oracle.decode_attention(qb, pool, bt, (pos + 1).astype(np.int32), scale)
        for b, r in enumerate(batch):
            where = (f"layer {l} request {r.id} ({ex.residency(r.id)[l]}) pos {pos[b]}: "
                     f"gpu nan {np.isnan(out[l, b]).any()} oracle nan {np.isnan(want[b]).any()}")
            np.testing.assert_allclose(out[l, b], want[b], rtol=RTOL, atol=ATOL, err_msg=where)


def test_engine_with_executor_is_bit_exact_and_correct():
    from paper_2601_10729_b200.executor import B200Executor, ModelShape

    prof = SystemProfile(num_layers=4, compute_base_ms=0.2, compute_per_token_ms=0.0004,
                         bandwidth_blocks_per_ms=12.0, gpu_block_budget=120, block_size=16,
                         prefill_per_token_ms=0.001)
    slo = SloConfig(tbt_target_ms=2.5, tpot_target_ms=2.5, window_min=2, window_max=6)
    trace = workload.Trace(tuple(workload.TraceRequest(i * 3, 90 + 37 * i, 6 + i % 3)
                                 for i in range(6)), {})
    cfg = RunConfig(max_batch=3)

    def run(executor):
        policy = make_policy(PolicyKind.ORBIT, prof, slo, max_batch=3, token_cap=cfg.batch_token_cap)
        sim = Simulation(trace, policy, prof, slo, cfg, executor=executor)
        return sim, sim.execute()

    _, ref_log = run(None)

    class Checked(B200Executor):
        steps_checked = 0

        def decode_step(self, batch, placement=None, inputs=None):
            ms = super().decode_step(batch, placement, inputs)
            for req, row in zip(batch, placement.rows):
                assert self.residency(req.id) == ["dev" if b else "host" for b in row]
            _check_step_outputs(self, batch)
            Checked.steps_checked += 1
            return ms

    ex = Checked.for_trace(trace, prof, shape=ModelShape(4, 8, 2), max_batch=3, record_timing=True)
    _, log = run(ex)
    stripped = [dict(r, payload={k: v for k, v in r["payload"].items() if k != "measured_us"})
                if r["kind"] == "step" else r for r in log]
    assert stripped == ref_log
    assert Checked.steps_checked == sum(1 for r in log if r["kind"] == "step")
    assert any(0 in row for r in log if r["kind"] == "step" for row in r["payload"]["rows"])
    assert ex.migrated["moves"] >= 0
    ex.close()


def test_cfg1_plan_fetch_volume_and_outputs():
    from paper_2601_10729_b200.executor import TOY

    batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=4088, target_output_tokens=64)
             for i in range(4)]
    placement = PlacementMatrix((0, 1, 2, 3), 4, ((0, 0, 0, 0), (0, 0, 0, 0), (1, 1, 1, 1), (1, 1, 1, 1)))
    ex = _executor(TOY, device_blocks=4 * 4 * 262 + 8 * 262, host_blocks=4 * 4 * 262 + 16,
                   record_timing=True)
    ex.install(batch, placement)
    for _ in range(3):
        ex.decode_step(batch, placement)
        _check_step_outputs(ex, batch)
        t = ex.last_timing
        assert t["copies"] == 8
        assert t["copy_bytes"] == blocks_to_fetch(placement, batch) * TOY.block_bytes
        for r in batch:
            r.record_generated_token()
    ex.close()


@pytest.mark.parametrize("slots", [1, 2])
def test_reconfiguration_round_trip_is_byte_exact(slots):
    from paper_2601_10729_b200.executor import ModelShape

    shape = ModelShape(6, 8, 2)
    batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=300 + 50 * i,
                          target_output_tokens=40) for i in range(3)]
    ex = _executor(shape, device_blocks=6 * 3 * 30 + 64, host_blocks=6 * 3 * 30 + 64,
                   staging_slots=slots)
    a = PlacementMatrix.from_strides([0, 1, 2], 6, [2, 3, None])
    b = PlacementMatrix.from_strides([0, 1, 2], 6, [3, None, 1])
    ex.install(batch, a)
    for _ in range(2):
        ex.decode_step(batch, a)
        for r in batch:
            r.record_generated_token()
    before = {(r.id, l): ex.slab_bits(r.id, l, r.blocks_per_layer) for r in batch for l in range(6)}
    ex.install(batch, b)          # evicts and restores layers (K4)
    ex.install(batch, a)          # and back
    after = {(r.id, l): ex.slab_bits(r.id, l, r.blocks_per_layer) for r in batch for l in range(6)}
    for key in before:
        np.testing.assert_array_equal(before[key], after[key])
    ex.decode_step(batch, a)
    _check_step_outputs(ex, batch)
    ex.close()


def test_pipelined_steps_match_synchronous_steps():
    """sync=False (host prepares step N+1 while the GPU runs N) gives bit-identical
    outputs, slabs and fetch accounting to step-by-step synchronous execution."""
    from paper_2601_10729_b200.executor import ModelShape

    shape = ModelShape(4, 8, 2)
    results = []
    for sync in (True, False):
        batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=200 + 91 * i,
                              target_output_tokens=32) for i in range(3)]
        ex = _executor(shape, device_blocks=400, host_blocks=400, record_timing=True, seed=5)
        pm = PlacementMatrix.from_strides([0, 1, 2], 4, [2, None, 1])
        ex.install(batch, pm)
        ex.runtime.timing_reset()
        outs = []
        for step in range(6):
            ex.decode_step(batch, pm, ex.synthetic_inputs(3, step=step), sync=sync)
            outs.append(ex.last_output)
            for r in batch:
                r.record_generated_token()
        ex.drain()
        tm = ex.runtime.timing()
        # valid token rows only: the tail of a slab's last block is never written
        slabs = []
        for r in batch:
            for l in range(4):
                bits = ex.slab_bits(r.id, l, r.blocks_per_layer)
                flat = bits.transpose(0, 3, 1, 2, 4).reshape(-1, *bits.shape[1:3], 128)
                slabs.append(flat[: r.total_tokens])
        results.append(([o.cpu() for o in outs], slabs, tm["acc_steps"], tm["acc_copy_bytes"]))
        ex.close()
    (o1, s1, n1, b1), (o2, s2, n2, b2) = results
    for a, b in zip(o1, o2):
        assert torch.equal(a, b)
    for a, b in zip(s1, s2):
        np.testing.assert_array_equal(a, b)
    assert n1 == n2 == 6 and b1 == b2


def test_tensor_parallel_split_step_matches_fused_step():
    """The per-layer split step (begin / layers(1) / end + o-proj per layer) used by
    the TP decoder produces bit-identical attention outputs to the one-call step,
    and its hidden state equals out @ W_o."""
    from paper_2601_10729_b200.executor import ModelShape
    from paper_2601_10729_b200.tp import HeadShard, TensorParallelDecoder

    shape = ModelShape(4, 8, 2)
    outs = []
    for split in (False, True):
        batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=150 + 80 * i,
                              target_output_tokens=16) for i in range(3)]
        ex = _executor(shape, device_blocks=300, host_blocks=300, seed=9)
        pm = PlacementMatrix.from_strides([0, 1, 2], 4, [2, None, 1])
        ex.install(batch, pm)
        inp = ex.synthetic_inputs(3, step=0)
        if split:
            tpd = TensorParallelDecoder(ex, HeadShard(0, 1, 8, 2), hidden=256, seed=1)
            hidden = tpd.step(batch, inp)
            ex.drain()
            want = torch.einsum("lbk,lhk->lbh", ex.last_output.reshape(4, 3, -1).float(),
                                tpd.w_o.float())
            torch.testing.assert_close(hidden.float(), want, rtol=2e-2, atol=2e-2)
        else:
            ex.decode_step(batch, pm, inp)
        outs.append(ex.last_output.clone())
        ex.close()
    assert torch.equal(outs[0], outs[1])


def test_live_mode_engine_runs_on_measured_time():
    from paper_2601_10729_b200.executor import B200Executor, ModelShape

    prof = SystemProfile(num_layers=4, compute_base_ms=0.05, compute_per_token_ms=1e-6,
                         bandwidth_blocks_per_ms=800.0, gpu_block_budget=150, block_size=16,
                         prefill_per_token_ms=0.0001)
    slo = SloConfig(tbt_target_ms=5.0, tpot_target_ms=5.0, window_min=2, window_max=6)
    trace = workload.Trace(tuple(workload.TraceRequest(i, 120 + 50 * i, 5) for i in range(4)), {})
    policy = make_policy(PolicyKind.ORBIT, prof, slo, max_batch=3)
    ex = B200Executor.for_trace(trace, prof, shape=ModelShape(4, 8, 2), max_batch=3)
    log = Simulation(trace, policy, prof, slo, RunConfig(max_batch=3), executor=ex,
                     mode="live").execute()
    steps = [r for r in log if r["kind"] == "step"]
    assert steps and all(r["payload"]["measured_us"] > 0 for r in steps)
    # the clock advanced by measured step times, not the model's
    from paper_2601_10729_b200.metrics import collect_metrics
    rep = collect_metrics(log)
    assert rep.requests_finished == 4 and rep.tokens_delivered == 20
    ex.close()


def test_bench_multi_rank_path_on_one_gpu():
    """torchrun N=2 through bench.py's TP path (KV-head shards, per-layer o-proj +
    all-reduce, max-over-ranks timing, rank-0 JSON) with gloo so both ranks can
    share the single GPU of this box - exercises the N>1 code the 8-GPU run uses."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, OFB_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29513", str(root / "bench.py"),
           "--gpus", "2", "--config", "cfg1", "--steps", "3", "--warmup", "3"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert "tp2" in line["config"]["parallelism"] and line["value"] > 0


def test_cli_simulate_on_b200_and_report_rerender(tmp_path):
    """`kvsim simulate --executor b200` runs every decode step on the GPU; its NDJSON
    event log (with measured_us per step) re-renders byte-stably via `report`."""
    from paper_2601_10729_b200.cli import main
    from paper_2601_10729_b200.metrics import load_log

    trace = tmp_path / "t.trace"
    assert main(["gen-trace", "--out", str(trace), "--rate", "400", "--seed", "3", "--count", "6",
                 "--prompt-median", "120", "--output-median", "8", "--max-prompt", "400",
                 "--max-output", "16"]) == 0
    report, log_path = tmp_path / "r.json", tmp_path / "run.log"
    assert main(["simulate", "--trace", str(trace), "--policy", "orbit", "--executor", "b200",
                 "--report", str(report), "--event-log", str(log_path)]) == 0
    steps = [r for r in load_log(log_path) if r["kind"] == "step"]
    assert steps and all("measured_us" in r["payload"] for r in steps)
    again = tmp_path / "again.json"
    assert main(["report", "--event-log", str(log_path), "--out", str(again)]) == 0
    assert again.read_bytes() == report.read_bytes()
    # decisions equal the model-only run of the same trace
    model_report = tmp_path / "m.json"
    assert main(["simulate", "--trace", str(trace), "--policy", "orbit", "--report",
                 str(model_report)]) == 0
    assert model_report.read_bytes() == report.read_bytes()


@pytest.mark.parametrize("policy", ["orbit", "dynamic_heuristic", "flexgen_plus", "deepspeed_like"])
def test_policies_with_deferral_and_preemption_under_executor(policy):
    """Tight budget: Orbit pauses/resumes (lazy eviction of removable layers, K4),
    baselines preempt (KV dropped, request re-prefilled on re-admission).  Decisions
    stay identical to the model-only run and residency equals the table each step."""
    from paper_2601_10729_b200.executor import B200Executor, ModelShape

    prof = SystemProfile(num_layers=6, compute_base_ms=0.3, compute_per_token_ms=0.002,
                         bandwidth_blocks_per_ms=4.0, gpu_block_budget=140, block_size=16,
                         prefill_per_token_ms=0.002)
    slo = SloConfig(tbt_target_ms=4.0, tpot_target_ms=4.0, window_min=2, window_max=6)
    trace = workload.Trace(tuple(workload.TraceRequest(i * 2, 150 + 45 * i, 4 + i % 4)
                                 for i in range(8)), {})
    cfg = RunConfig(max_batch=4)

    def run(executor):
        pol = make_policy(PolicyKind(policy), prof, slo, max_batch=4, token_cap=cfg.batch_token_cap)
        return Simulation(trace, pol, prof, slo, cfg, executor=executor).execute()

    ref = run(None)

    class Checked(B200Executor):
        def decode_step(self, batch, placement=None, inputs=None, sync=True):
            ms = super().decode_step(batch, placement, inputs, sync)
            for req, row in zip(batch, placement.rows):
                assert self.residency(req.id) == ["dev" if b else "host" for b in row]
            return ms

    ex = Checked.for_trace(trace, prof, shape=ModelShape(6, 8, 2), max_batch=4)
    log = run(ex)
    strip = [dict(r, payload={k: v for k, v in r["payload"].items() if k != "measured_us"})
             if r["kind"] == "step" else r for r in log]
    assert strip == ref
    kinds = {r["kind"] for r in ref}
    if policy == "orbit":
        assert "pause" in kinds or "replan" in kinds
    ex.close()


def test_reactive_preemption_releases_and_reprefills():
    """flexgen_like with a static stride that stops fitting: the engine preempts the
    youngest request (KV dropped, executor.release), re-admits and re-prefills it;
    decisions identical to the model-only run."""
    from paper_2601_10729_b200.executor import B200Executor, ModelShape
    from paper_2601_10729_b200.policies import PolicyOptions

    prof = SystemProfile(num_layers=6, compute_base_ms=0.3, compute_per_token_ms=0.002,
                         bandwidth_blocks_per_ms=4.0, gpu_block_budget=80, block_size=16,
                         prefill_per_token_ms=0.002)
    slo = SloConfig(tbt_target_ms=4.0, tpot_target_ms=4.0, window_min=2, window_max=6)
    trace = workload.Trace(tuple(workload.TraceRequest(i * 2, 150 + 45 * i, 4 + i % 4)
                                 for i in range(8)), {})
    opts = PolicyOptions(static_stride=None, worst_case_tokens=600)

    def run(executor):
        pol = make_policy(PolicyKind.FLEXGEN_LIKE, prof, slo, opts, max_batch=4)
        return Simulation(trace, pol, prof, slo, RunConfig(max_batch=4), executor=executor).execute()

    ref = run(None)
    assert sum(1 for r in ref if r["kind"] == "preempt") >= 1
    ex = B200Executor.for_trace(trace, prof, shape=ModelShape(6, 8, 2), max_batch=4)
    log = run(ex)
    strip = [dict(r, payload={k: v for k, v in r["payload"].items() if k != "measured_us"})
             if r["kind"] == "step" else r for r in log]
    assert strip == ref
    assert not ex.slabs            # everything released at the end
    ex.close()


@pytest.mark.parametrize("slots", [1, 2])
def test_cross_step_prefetch_is_invisible(slots):
    """Each step enqueues the next step's first fetches (cross-step prefetch); the
    next step adopts them when its plan is unchanged and fences them otherwise.
    Outputs must be bit-identical to running without it, across a plan change
    (migration + fence) and a released request."""
    from paper_2601_10729_b200.executor import ModelShape

    shape = ModelShape(6, 8, 2)
    runs = {}
    for prefetch in (False, True):
        batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=300 + 57 * i,
                              target_output_tokens=40) for i in range(3)]
        ex = _executor(shape, device_blocks=4000, host_blocks=4000, staging_slots=slots, seed=11,
                       prefetch_next=prefetch)
        pm = PlacementMatrix.from_strides([0, 1, 2], 6, [2, 1, None])
        ex.install(batch, pm)
        outs = []
        for step in range(9):
            if step == 4:      # plan change: restores + evictions, prefetch fenced
                pm = PlacementMatrix.from_strides([0, 1, 2], 6, [1, 2, 3])
                ex.install(batch, pm)
            if step == 7:      # request 2 leaves the batch
                ex.release(2)
                batch = batch[:2]
                pm = PlacementMatrix((0, 1), 6, pm.rows[:2])
            ex.decode_step(batch, pm, ex.synthetic_inputs(len(batch), step=step))
            outs.append(ex.last_output.clone())
            if step in (3, 8):
                _check_step_outputs(ex, batch)
            for r in batch:
                r.record_generated_token()
        runs[prefetch] = (outs, ex.runtime.prefetch_stats())
        ex.close()
    for a, b in zip(runs[False][0], runs[True][0]):
        assert torch.equal(a, b)
    assert runs[False][1]["adopted"] == 0
    assert runs[True][1]["adopted"] >= 5, runs[True][1]


def test_cross_step_prefetch_in_the_tensor_parallel_split_step():
    """The per-layer split step (TP decoder: K1 + K6 per layer) adopts the cross-step
    prefetch too; hidden states are bit-identical with and without it."""
    from paper_2601_10729_b200.executor import ModelShape
    from paper_2601_10729_b200.tp import HeadShard, TensorParallelDecoder

    shape = ModelShape(4, 8, 2)
    hiddens, stats = {}, {}
    for prefetch in (False, True):
        batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=200 + 90 * i,
                              target_output_tokens=16) for i in range(3)]
        ex = _executor(shape, device_blocks=2000, host_blocks=2000, staging_slots=2, seed=4,
                       prefetch_next=prefetch)
        pm = PlacementMatrix.from_strides([0, 1, 2], 4, [2, 1, None])
        ex.install(batch, pm)
        tpd = TensorParallelDecoder(ex, HeadShard(0, 1, 8, 2), hidden=256, seed=2, max_batch=3)
        out = []
        for step in range(4):
            out.append(tpd.step(batch, ex.synthetic_inputs(3, step=step)).clone())
            for r in batch:
                r.record_generated_token()
        ex.drain()
        hiddens[prefetch] = [h.cpu() for h in out]
        stats[prefetch] = ex.runtime.prefetch_stats()
        tpd.close()
        ex.close()
    for a, b in zip(hiddens[False], hiddens[True]):
        assert torch.equal(a, b)
    assert stats[True]["adopted"] == 3 and stats[False]["adopted"] == 0


def test_live_calibration_of_the_cost_model():
    """the SystemProfile the planner prices with can be measured on the
    box (K1 slope / intercept, pinned link) instead of taken from constants."""
    from paper_2601_10729_b200.calibrate import measure_b200_profile

    # contexts large enough that the slope is the streaming rate, not launch latency
    prof, raw = measure_b200_profile(32, 32, 8, 100_000, batch=8, contexts=(4096, 32768), iters=5)
    assert 3000 < raw["k1_gbs_slope"] < 9000, raw
    assert 0.0 <= raw["layer_fixed_ms"] < 0.1, raw
    assert 30 < raw["h2d_gbs"] < 70, raw
    assert prof.num_layers == 32 and prof.gpu_block_budget == 100_000
    assert prof.bandwidth_blocks_per_ms == pytest.approx(raw["h2d_gbs"] * 1e6 / 65536)


@pytest.mark.parametrize("hq,hkv", [(16, 1), (4, 4), (64, 8)])
def test_full_step_other_head_layouts(hq, hkv):
    """The whole step (K3 append, K2 fetches, K1) for GQA group 16, MHA (group 1)
    and the 70B head layout, vs the oracle on every (layer, request)."""
    from paper_2601_10729_b200.executor import ModelShape

    shape = ModelShape(4, hq, hkv)
    batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=130 + 77 * i,
                          target_output_tokens=8) for i in range(3)]
    pm = PlacementMatrix.from_strides([0, 1, 2], 4, [2, None, 1])
    ex = _executor(shape, device_blocks=400, host_blocks=400, staging_slots=2, seed=hq + hkv)
    try:
        ex.install(batch, pm)
        for _ in range(2):
            ex.decode_step(batch, pm)
            _check_step_outputs(ex, batch)
            for r in batch:
                r.record_generated_token()
    finally:
        ex.close()


@pytest.mark.parametrize("mode", ["auto", "bal", "split"])
@pytest.mark.parametrize("heads,B,ctx", [((32, 8), 1, 4096), ((32, 8), 2, 1500), ((8, 1), 3, 2900),
                                         ((32, 8), 4, 1024)])
def test_attention_only_steps_late_wait_and_balanced_plan(monkeypatch, heads, B, ctx, mode):
    """All-resident steps (every layer but the first launched kv_ready: K1's consumers
    wait for the previous layer only before their global writes) on the balanced narrow
    plan, the cost-model plan and the auto policy: every layer of several consecutive
    steps equals the oracle (profiles/r02_k1_instep.md)."""
    from paper_2601_10729_b200 import _native
    from paper_2601_10729_b200.executor import ModelShape

    if mode == "auto":
        monkeypatch.delenv("OFB_K1_INSTEP", raising=False)
    else:
        monkeypatch.setenv("OFB_K1_INSTEP", mode)
    hq, hkv = heads
    shape = ModelShape(4, hq, hkv)
    batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=ctx - 53 * i, target_output_tokens=16)
             for i in range(B)]
    cap = -(-(ctx + 20) // 16)
    ex = _executor(shape, device_blocks=B * 4 * cap + 16, host_blocks=16)
    ex.install(batch, PlacementMatrix.from_strides(range(B), 4, [None] * B))
    if mode == "bal" and B == 1 and hkv == 8:   # the plan this case exists for
        import ctypes
        bps, ns, narrow = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        assert _native.load().ofb_attention_instep_plan(B, hq, hkv, ctx + 1, 148, 3, ctypes.byref(bps),
                                                        ctypes.byref(ns), ctypes.byref(narrow)) == 0
        assert narrow.value == 1 and ns.value * hkv * B <= 148
    for _ in range(3):
        ex.decode_step(batch, None, None, sync=True)
        _check_step_outputs(ex, batch)
        for r in batch:
            r.record_generated_token()
    ex.close()
