"""Multi-process (world_size 2, gloo, CPU) tests of the tensor-parallel host
logic: KV-head sharding, the C1 o-projection all-reduce and C2 plan
replication.  The GPU side uses the same functions over NCCL."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_10729_b200.tp import HeadShard, check_plan_replicated, oproj_allreduce, shard_oproj


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as exc:  # pragma: no cover - surfaced in the parent
        q.put((rank, f"error: {exc!r}"))
    finally:
        dist.destroy_process_group()


def _run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    return out


def test_head_shard_ranges():
    s = [HeadShard(r, 4, 64, 8) for r in range(4)]
    assert [list(x.kv_heads) for x in s] == [[0, 1], [2, 3], [4, 5], [6, 7]]
    assert s[1].q_heads == range(16, 32) and s[1].local_q == 16 and s[1].local_kv == 2
    # every query head's KV head is owned by the same rank (GQA group stays local)
    for x in s:
        assert {h // 8 for h in x.q_heads} == set(x.kv_heads)
    with pytest.raises(ValueError):
        HeadShard(0, 3, 64, 8)


def _oproj_case(rank, world):
    g = torch.Generator().manual_seed(0)
    B, hq, hkv, hidden = 3, 8, 2, 64
    attn = torch.randn((B, hq, 128), generator=g)
    w_o = torch.randn((hq * 128, hidden), generator=g)
    shard = HeadShard(rank, world, hq, hkv)
    local = attn[:, shard.q_heads.start: shard.q_heads.stop].contiguous()
    got = oproj_allreduce(local, shard_oproj(w_o, shard))
    want = attn.reshape(B, -1) @ w_o
    return float((got - want).abs().max())


def test_oproj_allreduce_equals_full_projection():
    errs = _run(_oproj_case)
    assert all(isinstance(e, float) and e < 1e-3 for e in errs.values()), errs


def _plan_case(rank, world):
    from paper_2601_10729_b200.core import RequestState, SloConfig, SystemProfile
    from paper_2601_10729_b200.planner import solve

    prof = SystemProfile(8, 0.5, 0.0005, 10.0, 200, 16)   # forces a mixed offload plan
    slo = SloConfig(50.0, 50.0, window_min=2, window_max=8)
    batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=100 + 60 * i,
                          target_output_tokens=50) for i in range(3)]
    rows = solve(batch, prof, slo, 1).placement.rows
    assert any(0 in r for r in rows) and any(1 in r for r in rows)
    same = check_plan_replicated(rows)
    perturbed = [list(r) for r in rows]
    if rank == 1:
        perturbed[0][0] ^= 1
    differ = check_plan_replicated(perturbed)
    return same, differ


def test_plans_are_replicated_across_ranks():
    res = _run(_plan_case)
    assert all(v == (True, False) for v in res.values()), res
