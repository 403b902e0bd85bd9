"""Tensor parallelism for the data path: KV-head sharding + C1 / C2.

SURVEY.md 8(e): attention of a (request, layer, KV head) touches only that
head's KV (GQA), so rank g of N owns KV heads
[g*Hkv/N, (g+1)*Hkv/N) and their Hq/N query heads for every request and
layer; each rank streams its own shard of offloaded KV over its own host
link.  The exchange a TP decoder really has follows attention: the
o-projection of the local heads yields a partial [B, hidden] that is summed
across ranks (C1, one all-reduce per layer; 512 KiB at 70B B=32).  Plans are
pure functions of the batch, so every rank recomputes the identical
placement (C2) - ``check_plan_replicated`` verifies it with one tiny
all-gather instead of broadcasting B x L bits every step.

On the GPU the exchange is K6 (``collective.py``: tcgen05 projection fused
with a one-shot all-reduce over IPC peer memory); ``oproj_allreduce`` below is
the same C1 written with ``torch.distributed`` - the formulation the gloo
host-logic tests check and the plain reference the kernel is compared with.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class HeadShard:
    """Which heads a rank owns."""

    rank: int
    world: int
    num_q_heads: int
    num_kv_heads: int

    def __post_init__(self) -> None:
        if self.num_kv_heads % self.world:
            raise ValueError(f"{self.num_kv_heads} KV heads do not shard over {self.world} ranks")
        if self.num_q_heads % self.num_kv_heads:
            raise ValueError("Hq must be a multiple of Hkv")
        if not 0 <= self.rank < self.world:
            raise ValueError("rank out of range")

    @property
    def kv_heads(self) -> range:
        n = self.num_kv_heads // self.world
        return range(self.rank * n, (self.rank + 1) * n)

    @property
    def q_heads(self) -> range:
        n = self.num_q_heads // self.world
        return range(self.rank * n, (self.rank + 1) * n)

    @property
    def local_q(self) -> int:
        return self.num_q_heads // self.world

    @property
    def local_kv(self) -> int:
        return self.num_kv_heads // self.world


def shard_oproj(w_o_full: torch.Tensor, shard: HeadShard, head_dim: int = 128) -> torch.Tensor:
    """Rows of W_o [Hq*d, hidden] that multiply this rank's heads' outputs."""
    lo = shard.q_heads.start * head_dim
    hi = shard.q_heads.stop * head_dim
    return w_o_full[..., lo:hi, :].contiguous()


def oproj_allreduce(attn_local: torch.Tensor, w_o_local: torch.Tensor, group=None) -> torch.Tensor:
    """C1: hidden = sum over ranks of attn_local [B, Hq/N, d] @ W_o_local [Hq/N*d, hidden]."""
    import torch.distributed as dist

    b = attn_local.shape[0]
    partial = attn_local.reshape(b, -1) @ w_o_local
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(partial, group=group)
    return partial


def check_plan_replicated(rows, group=None) -> bool:
    """C2: every rank computed the same placement rows (one all-gather of a digest)."""
    import hashlib

    import torch.distributed as dist

    digest = hashlib.sha256(repr(tuple(tuple(r) for r in rows)).encode()).digest()[:8]
    mine = torch.tensor([int.from_bytes(digest, "little", signed=True)], dtype=torch.int64)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return True
    if dist.get_backend(group) == "nccl":
        mine = mine.cuda()
    gathered = [torch.zeros_like(mine) for _ in range(dist.get_world_size(group))]
    dist.all_gather(gathered, mine, group=group)
    return all(int(g.item()) == int(mine.item()) for g in gathered)


class TensorParallelDecoder:
    """One rank of a KV-head-sharded decode step: the executor's native step
    split per layer, each layer followed by the fused o-projection + all-reduce
    (K6, ``collective.OprojAllReduce``) on the same stream, so layer l+1 is
    ordered after layer l's exchange - the dependency a real decoder has (q of
    l+1 derives from hidden of l).  With ``torch.distributed`` initialised and
    world > 1 the ranks exchange CUDA IPC handles once and the kernel pushes
    its tiles straight into the peers' memory; otherwise it is the projection
    alone (a TP-N shard emulated on one GPU)."""

    def __init__(self, executor, shard: HeadShard, hidden: int, group=None, seed: int = 0,
                 max_batch: int = 256):
        import torch.distributed as dist

        from .collective import OprojAllReduce, SymmetricBuffers

        self.ex = executor
        self.shard = shard
        self.hidden = hidden
        self.group = group
        L = executor.shape.num_layers
        g = torch.Generator(device=executor.device)
        g.manual_seed(1234 + seed)   # identical full W_o on every rank; each keeps its columns
        full_k = shard.num_q_heads * 128
        lo, hi = shard.q_heads.start * 128, shard.q_heads.stop * 128
        scale = full_k ** -0.5
        # nn.Linear layout [hidden, Hq*128]; this rank multiplies its heads' columns
        w_o = torch.empty((L, hidden, hi - lo), dtype=torch.bfloat16, device=executor.device)
        for l in range(L):
            w = torch.randn((hidden, full_k), generator=g, device=executor.device) * scale
            w_o[l] = w[:, lo:hi].to(torch.bfloat16)
        world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        self.symm = None
        if world > 1:
            if world != shard.world:
                raise ValueError("process group size differs from the head shard's world")
            self.symm = SymmetricBuffers(world, shard.rank, max_batch, hidden, group=group,
                                         device=executor.device)
        self.proj = OprojAllReduce(w_o, max_batch, self.symm)   # keeps only the packed copy
        del w_o
        self.last_hidden = None

    @property
    def w_o(self) -> torch.Tensor:
        """This rank's W_o rows [L, hidden, Hq_local*128] (Linear layout), unpacked."""
        w = self.proj.w
        if self.proj.w_layout == 0:
            return w
        L, tiles, chunks = w.shape[:3]
        return w.permute(0, 1, 3, 2, 4).reshape(L, tiles * 128, chunks * 64)

    def step(self, batch, inputs=None) -> torch.Tensor:
        ex = self.ex
        desc, keep = ex.prepare_step(batch, inputs)
        stream = torch.cuda.current_stream()
        L, B = ex.shape.num_layers, len(batch)
        out = keep[1]
        hidden = torch.empty((L, B, self.hidden), dtype=torch.bfloat16, device=ex.device)
        ex.runtime.step_begin(desc, stream)
        try:
            for l in range(L):
                ex.runtime.step_layers(1)
                self.proj(out, l, out=hidden[l], stream=stream)
        except BaseException:
            ex.runtime.step_abort()   # the original error propagates, not a step_end one
            raise
        ex.runtime.step_end()
        done = torch.cuda.Event()
        done.record(stream)
        ex.steps += 1
        ex.last_inputs, ex.last_output = keep[0], out
        ex._inflight.append((done, (keep, hidden)))
        while len(ex._inflight) > 3:
            ex._inflight.popleft()[0].synchronize()
        self.last_hidden = hidden
        return hidden

    def close(self) -> None:
        if self.symm is not None:
            self.symm.check()
            self.symm.close()
            self.symm = None
