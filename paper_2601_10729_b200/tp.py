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


def _world(group) -> int:
    import torch.distributed as dist

    return dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1


class TensorParallelLlama:
    """One rank of a whole Llama decoder step, KV-head sharded.

    Per layer, on one stream: input RMSNorm -> q / k / v projections of this
    rank's heads -> K3 append of the fresh token + K2 fetch wait + K1
    attention (the native step split per layer, ``append_per_layer``: k_new /
    v_new of layer l only exist once layer l-1 finished) -> o-projection with
    its all-reduce (C1) -> residual -> RMSNorm -> gate / up projection (cuBLAS)
    -> SiLU * up -> down projection with its all-reduce -> residual.  So every
    weight byte of the 70B shard is streamed from HBM each step (137 GB / TP),
    and the step time is the real decoder's, not attention alone.

    ``c1="k6"``: every projection is K6 (``collective.OprojAllReduce``: tcgen05
    projection, the o / down ones fused with the one-shot all-reduce over IPC
    peer memory) and the glue is folded into it: each RMSNorm becomes the
    producing K6's per-tile row sum of squares (``ss_out``, after the residual
    add) plus a 1/rms row scale in the consuming K6's epilogue (``ss_in``; the
    norm weight is folded into its packed W), and SwiGLU is the gate/up K6's
    epilogue (gate/up rows interleaved per 64) - 3 launches fewer per layer.
    ``c1="nccl"``: cuBLAS
    projection + ``torch.distributed.all_reduce`` (NCCL over NVLink) - the
    unfused baseline the north star names.  With world 1 (a
    TP-N shard emulated on one GPU) there is no exchange in either arm.
    Weights are random bf16 (no checkpoint), scaled 1/sqrt(fan_in); norms are
    unit-weight.
    """

    def __init__(self, executor, shard: HeadShard, hidden: int, intermediate: int, *,
                 c1: str = "k6", group=None, seed: int = 0, max_batch: int = 256,
                 eps: float = 1e-5):
        from .collective import OprojAllReduce, SymmetricBuffers

        if c1 not in ("k6", "nccl"):
            raise ValueError("c1 must be 'k6' or 'nccl'")
        if intermediate % shard.world:
            raise ValueError("intermediate size must divide by the TP degree")
        ex = self.ex = executor
        self.shard, self.hidden, self.group, self.c1, self.eps = shard, hidden, group, c1, eps
        L, dev = ex.shape.num_layers, ex.device
        hq, hkv = shard.local_q, shard.local_kv
        self.inter = intermediate // shard.world
        self.world = _world(group)
        if self.world > 1 and self.world != shard.world:
            raise ValueError("process group size differs from the head shard's world")
        g = torch.Generator(device=dev)
        g.manual_seed(7001 + 131 * seed + shard.rank)

        from .collective import interleave_gate_up, pack_weight

        self.norm = torch.ones((2, hidden), dtype=torch.bfloat16, device=dev)

        def rand(shape, fan_in, packed=False, norm=None, gate_up=False):
            """Random bf16 layers, generated one layer at a time (no full-size
            temporaries: the 70B shard fills most of HBM); ``packed``: K6 layout,
            with ``norm`` (the input RMSNorm weight) folded into the columns and
            ``gate_up`` rows interleaved for the SwiGLU epilogue."""
            L_, h, k = shape
            out = torch.empty((L_, h // 128, k // 64, 128, 64) if packed else shape,
                              dtype=torch.bfloat16, device=dev)
            for l in range(L_):
                w = (torch.randn((h, k), generator=g, device=dev) * fan_in ** -0.5).to(torch.bfloat16)
                if packed:
                    if norm is not None:
                        w = (w.float() * norm.float()[None, :]).to(torch.bfloat16)
                    if gate_up:
                        w = interleave_gate_up(w)
                    w = pack_weight(w)
                out[l] = w
            return out

        qkv_rows = (hq + 2 * hkv) * 128
        packed = c1 == "k6"
        # with K6 every projection runs on it (the column-parallel q/k/v and
        # gate/up ones with world 1: no exchange); the NCCL arm is the cuBLAS
        # baseline throughout
        self.w_qkv = rand((L, qkv_rows, hidden), hidden, packed, norm=self.norm[0])
        self.w_gu = rand((L, 2 * self.inter, hidden), hidden, packed, norm=self.norm[1], gate_up=True)
        if packed:
            self.qkv_proj = OprojAllReduce(self.w_qkv, max_batch)
            self.gu_proj = OprojAllReduce(self.w_gu, max_batch)
        w_o = rand((L, hidden, hq * 128), shard.num_q_heads * 128, packed)
        w_d = rand((L, hidden, self.inter), intermediate, packed)
        self.symm = None
        if c1 == "k6":
            if self.world > 1:
                self.symm = SymmetricBuffers(self.world, shard.rank, max_batch, hidden, group=group,
                                             device=dev)
            self.oproj = OprojAllReduce(w_o, max_batch, self.symm)
            self.down = OprojAllReduce(w_d, max_batch, self.symm)
            del w_o, w_d
        else:
            self.w_o, self.w_d = w_o, w_d
        self.max_batch = max_batch
        self._bufs = None
        self._bufs_by_b = {}         # batch size -> step buffers
        self._k6_descs = {}          # (B, x parity) -> per layer prebuilt K6 descriptors
        self.last_hidden = None

    def layer_weights(self, l: int) -> dict:
        """Layer ``l``'s weights in ``nn.Linear`` layout [out, in] (test / reference use)."""
        nq, nk = self.shard.local_q * 128, self.shard.local_kv * 128

        from .collective import deinterleave_gate_up

        def unpack(t):
            if t.dim() == 2:
                return t
            tiles, chunks = t.shape[:2]
            return t.permute(0, 2, 1, 3).reshape(tiles * 128, chunks * 64)

        w, gu = unpack(self.w_qkv[l]), unpack(self.w_gu[l])
        if self.c1 == "k6":   # packed: gate/up interleaved, norm weights folded in (unit here)
            gu = deinterleave_gate_up(gu)
        o = unpack(self.oproj.w[l]) if self.c1 == "k6" else self.w_o[l]
        d = unpack(self.down.w[l]) if self.c1 == "k6" else self.w_d[l]
        return {"q": w[:nq], "k": w[nq:nq + nk], "v": w[nq + nk:], "o": o,
                "gate": gu[: self.inter], "up": gu[self.inter:], "down": d}

    @property
    def weight_bytes(self) -> int:
        """Bytes of weights one step streams (every layer's projections)."""
        L = self.ex.shape.num_layers
        per_layer = ((self.w_qkv[0].numel() + self.w_gu[0].numel())
                     + self.hidden * (self.shard.local_q * 128 + self.inter)) * 2
        return L * per_layer

    def _buffers(self, B: int):
        """Step buffers for batch size B, kept per B (a serving run cycles through a
        few batch sizes; the K6 descriptors point into them)."""
        bufs = self._bufs_by_b.get(B)
        if bufs is None:
            L, dev = self.ex.shape.num_layers, self.ex.device
            hq, hkv = self.shard.local_q, self.shard.local_kv
            mk = lambda *s: torch.empty(s, dtype=torch.bfloat16, device=dev)  # noqa: E731
            bufs = {"B": B, "q": mk(L, B, hq, 128), "k_new": mk(L, B, hkv, 128),
                    "v_new": mk(L, B, hkv, 128), "act": mk(L, B, self.inter),
                    "x": [mk(B, self.hidden), mk(B, self.hidden)], "attn_out": mk(L, B, hq, 128),
                    # per hidden tile, per row: sum of x^2 (the fused RMSNorms)
                    "ss": torch.empty((self.hidden // 128, self.max_batch), dtype=torch.float32,
                                      device=dev)}
            if self.c1 != "k6":   # the cuBLAS + NCCL arm's standalone glue buffers
                bufs.update({"h": mk(B, self.hidden), "a": mk(L, B, self.hidden),
                             "a2": mk(L, B, self.hidden), "gu": mk(B, 2 * self.inter)})
            self._bufs_by_b[B] = bufs
        self._bufs = bufs
        return bufs

    def _k6_plan(self, B: int, bufs: dict, parity: int) -> list:
        """Per layer, the four K6 descriptors of the fused step, built (and
        validated) once per batch size and residual buffer: a step then only
        patches this step's pool tables / positions into the q/k/v one and
        launches (host enqueue of a 70B TP8 step 5.4 -> 1.8 ms, against a 6.4 ms
        GPU step at 4K context)."""
        key = (B, parity)
        plan = self._k6_descs.get(key)
        if plan is not None:
            return plan
        x = bufs["x"][parity]
        q, kn, vn, ss = bufs["q"], bufs["k_new"], bufs["v_new"], bufs["ss"]
        nq, nk = self.shard.local_q * 128, self.shard.local_kv * 128
        kv0 = {"pool": 1, "tables": 1, "positions": 1, "host_slabs": 0, "max_blocks": 1, "part": 1,
               "block_bytes": self.ex.shape.block_bytes}      # patched every step
        # layer 0 through the validating path; the other layers are copies with
        # their layer index and per-layer output pointers patched (~1 ms a plan,
        # so a new batch size costs little inside a timed step)
        qkv0, _ = self.qkv_proj.prepare(x, 0, ss_in=ss, eps=self.eps, kv_append=kv0,
                                        parts=[q[0].view(B, nq), kn[0].view(B, nk), vn[0].view(B, nk)])
        o0, _ = self.oproj.prepare(bufs["attn_out"], 0, out=x, residual=x, ss_out=ss)   # C1
        gu0, _ = self.gu_proj.prepare(x, 0, out=bufs["act"][0], ss_in=ss, eps=self.eps, swiglu=True)
        dn0, _ = self.down.prepare(bufs["act"], 0, out=x, residual=x, ss_out=ss)
        plan = [(qkv0, o0, gu0, dn0)]
        copy = lambda d: type(d).from_buffer_copy(d)  # noqa: E731
        for l in range(1, self.ex.shape.num_layers):
            qkv, o, gu, dn = copy(qkv0), copy(o0), copy(gu0), copy(dn0)
            qkv.layer = o.layer = gu.layer = dn.layer = l
            qkv.part_out[0], qkv.part_out[1], qkv.part_out[2] = (q[l].data_ptr(), kn[l].data_ptr(),
                                                                 vn[l].data_ptr())
            gu.out = bufs["act"][l].data_ptr()
            plan.append((qkv, o, gu, dn))
        self._k6_descs[key] = plan
        return plan

    def _reduce(self, w, x_all, l, x, h):
        """The cuBLAS + NCCL arm of C1: x += sum over ranks of x_all[l] @ w[l]^T
        (projected into ``h``, all-reduced, added).  The K6 arm does this in one
        kernel with the residual add in its epilogue (``_k6_plan``)."""
        torch.matmul(x_all[l].reshape(h.shape[0], -1), w[l].t(), out=h)
        if self.world > 1:
            import torch.distributed as dist

            dist.all_reduce(h, group=self.group)
        x.add_(h)

    def _rmsnorm(self, x, weight, out, stream):
        from . import _native

        _native.check(_native.load().ofb_rmsnorm(x.data_ptr(), weight.data_ptr(), out.data_ptr(),
                                                 x.shape[0], self.hidden, float(self.eps),
                                                 stream.cuda_stream), "ofb_rmsnorm")

    def _silu_mul(self, gu, act, stream):
        from . import _native

        _native.check(_native.load().ofb_silu_mul(gu.data_ptr(), act.data_ptr(), gu.shape[0],
                                                  self.inter, stream.cuda_stream), "ofb_silu_mul")

    def step(self, batch, x_in: torch.Tensor) -> torch.Tensor:
        """One decode step of the whole decoder; ``x_in`` bf16 [B, hidden] (the
        new tokens' embeddings).  Returns the final hidden state [B, hidden]."""

        ex = self.ex
        B, L = len(batch), ex.shape.num_layers
        if B > self.max_batch:
            raise ValueError("batch exceeds max_batch")
        bufs = self._buffers(B)
        q, kn, vn = bufs["q"], bufs["k_new"], bufs["v_new"]
        desc, keep = ex.prepare_step(batch, {"q": q, "k_new": kn, "v_new": vn, "out": bufs["attn_out"]})
        k6 = self.c1 == "k6"
        # K6 writes the resident rows' new K/V straight into the pool (K3 folded
        # into the q/k/v epilogue); the runtime appends only host-slab rows
        desc.append_per_layer = 2 if k6 else 1
        out = keep[1]
        stream = torch.cuda.current_stream()
        x = bufs["x"][ex.steps % 2]
        x.copy_(x_in)
        h = bufs.get("h")
        nq, nk = self.shard.local_q * 128, self.shard.local_kv * 128
        a_all, a2_all, gu = bufs.get("a"), bufs.get("a2"), bufs.get("gu")
        ss = bufs["ss"]
        bt_layer = B * desc.max_blocks * 4
        sh = stream.cuda_stream
        plan = None
        if k6:   # the first layer's fused RMSNorm: row sums of squares of the embeddings
            from . import _native

            _native.check(_native.load().ofb_row_sumsq(x.data_ptr(), ss.data_ptr(), B, self.hidden,
                                                       self.max_batch, sh), "ofb_row_sumsq")
            plan = self._k6_plan(B, bufs, ex.steps % 2)
        ex.runtime.step_begin(desc, stream)
        try:
            for l in range(L):
                if k6:     # RMSNorm(x) . W_qkv^T for this rank's heads in one launch, into their
                    # buffers, the new token's K/V also into its pool slot (resident rows)
                    qd = plan[l][0]
                    qd.kv_pool, qd.kv_max_blocks = desc.kv_pool, desc.max_blocks
                    qd.kv_tables = desc.block_tables + l * bt_layer
                    qd.kv_positions = desc.positions
                    qd.kv_host_slabs = desc.host_slabs_dev + l * B * 8
                    self.qkv_proj.launch(qd, sh)
                else:
                    a = a_all[l]
                    self._rmsnorm(x, self.norm[0], a, stream)
                    w = self.w_qkv[l]
                    torch.matmul(a, w[:nq].t(), out=q[l].view(B, nq))
                    torch.matmul(a, w[nq:nq + nk].t(), out=kn[l].view(B, nk))
                    torch.matmul(a, w[nq + nk:].t(), out=vn[l].view(B, nk))
                ex.runtime.step_layers(1)                    # K3 + K2 wait + K1 of layer l
                if k6:
                    self.oproj.launch(plan[l][1], sh)         # x += o_proj(attn) (C1)
                    self.gu_proj.launch(plan[l][2], sh)       # act = silu(gate) * up of RMSNorm(x) . W_gu^T
                    self.down.launch(plan[l][3], sh)          # x += down(act) (C1)
                    continue
                # cuBLAS + NCCL arm: standalone glue between the projections
                self._reduce(self.w_o, out, l, x, h)                 # x += o_proj(attn) (C1)
                a2 = a2_all[l]
                self._rmsnorm(x, self.norm[1], a2, stream)
                torch.matmul(a2, self.w_gu[l].t(), out=gu)
                self._silu_mul(gu, bufs["act"][l], stream)
                self._reduce(self.w_d, bufs["act"], l, x, h)         # x += down(act) (C1)
        except BaseException:
            ex.runtime.step_abort()
            raise
        ex.runtime.step_end()
        done = torch.cuda.Event()
        done.record(stream)
        ex.steps += 1
        ex.last_inputs, ex.last_output = {"q": q, "k_new": kn, "v_new": vn}, out
        ex._inflight.append((done, keep))
        while len(ex._inflight) > 3:
            ex._inflight.popleft()[0].synchronize()
        self.last_hidden = x
        return x

    def close(self) -> None:
        if self.symm is not None:
            self.symm.check()
            self.symm.close()
            self.symm = None


class TensorParallelExecutor:
    """The engine seam (``sync_table`` / ``decode_step`` / ``release``, as
    ``executor.B200Executor``) for one rank of a KV-head-sharded deployment, so
    ``engine.Simulation`` drives a TP run (src/engine.py:708-734).

    Every rank runs its own engine; plans are pure functions of the batch
    (S:254), so the ranks compute the same placement (C2) - verified with one
    digest all-gather whenever the placement changes.  A step
    lasts as long as its slowest rank, so the device time a live clock sees is
    the max over ranks (one tiny all-reduce), which keeps the ranks' engines in
    lock step in every clock mode."""

    def __init__(self, decoder: TensorParallelLlama, group=None, seed: int = 0):
        self.dec = decoder
        self.ex = decoder.ex
        self.group = group
        self.seed = seed
        self.world = _world(group)
        self._rows = None
        self.steps = 0
        self.last_ms = None

    @property
    def prefill_wall_ms(self) -> float:
        return self.ex.prefill_wall_ms

    @property
    def migrated(self):
        return self.ex.migrated

    @property
    def runtime(self):
        return self.ex.runtime

    def sync_table(self, table, batch, paused=()) -> None:
        self.ex.sync_table(table, batch, paused)

    def release(self, rid: int) -> None:
        self.ex.release(rid)

    def embeddings(self, B: int) -> torch.Tensor:
        """Seeded stand-in for this step's token embeddings (same on every rank)."""
        g = torch.Generator(device=self.ex.device)
        g.manual_seed(90001 + 7919 * self.seed + self.steps)
        return torch.randn((B, self.dec.hidden), generator=g, device=self.ex.device).to(
            torch.bfloat16)

    def decode_step(self, batch, placement=None) -> float:
        ex = self.ex
        if placement is not None:
            rows = tuple(tuple(r) for r in placement.rows)
            if rows != self._rows:
                if not check_plan_replicated(rows, self.group):
                    raise RuntimeError("ranks computed different placements (C2 violated)")
                self._rows = rows
            for req, row in zip(batch, placement.rows):
                st = ex.slabs.get(req.id)
                if st is None or any((st.dev[l] is not None) != bool(b) for l, b in enumerate(row)):
                    raise RuntimeError("physical residency does not match the placement")
        x0 = self.embeddings(len(batch))
        stream = torch.cuda.current_stream()
        t1 = torch.cuda.Event(enable_timing=True)
        if ex._mig_start is not None:      # the step also waits for its plan's migration
            t0, ex._mig_start = ex._mig_start, None
        else:
            t0 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
        self.dec.step(batch, x0)
        t1.record(stream)
        t1.synchronize()
        ex._inflight.clear()
        self.steps += 1
        ms = t0.elapsed_time(t1)
        if self.world > 1:
            import torch.distributed as dist

            t = torch.tensor([ms], dtype=torch.float64)
            if dist.get_backend(self.group) == "nccl":
                t = t.to(ex.device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
            ms = float(t.item())
        self.last_ms = ms
        return ms

    def close(self) -> None:
        self.dec.close()
        self.ex.close()
