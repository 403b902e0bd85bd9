"""B200 executor: the physical side of the KV manager and of every decode step.

The engine (``engine.Simulation``) keeps the reference's bookkeeping - the
BlockTable's 'g' / 'h' / 'r' location per (request, layer)
(/root/reference/pkg/src/kvsim/engine.py:126-248).  This executor makes
that table true in memory and runs the step the reference only prices:

* ``sync_table``   after every ``apply_plan``: new requests get their
                   prefill KV written straight to the planned location
                   (S:421); host->GPU flips are H2D restores, GPU->host flips
                   (plan refinement or lazy eviction of a paused request's
                   removable layers) are D2H evictions - K4, batched on the
                   runtime's migration streams.
* ``decode_step``  appends the new token (K3), streams every offloaded slab
                   into its request's staging slot under the reference launch
                   rule (K2), and runs paged GQA attention per layer (K1) -
                   one native call, ``ofb_runtime_decode_step``.
* ``release``      frees a finished / preempted request's slabs.

KV values are synthetic (seeded N(0,1) bf16): there is no model checkpoint.
"""

from __future__ import annotations

import math
import time
from collections import deque
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from .core import PlacementMatrix, RequestState, blocks_for_tokens
from .kvpool import BLOCK_TOKENS, HEAD_DIM, DevicePool, HostArena
from .runtime import StepRuntime

_DEVICE_LOCS = ("g", "r")


@dataclass(frozen=True)
class ModelShape:
    """Attention geometry of the served model (per GPU shard)."""

    num_layers: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int = HEAD_DIM

    def __post_init__(self) -> None:
        if self.head_dim != HEAD_DIM:
            raise ValueError("head_dim must be 128")
        if self.num_q_heads % self.num_kv_heads or self.num_q_heads // self.num_kv_heads > 16:
            raise ValueError("Hq must be a multiple of Hkv with q-group <= 16")

    @property
    def block_bytes(self) -> int:
        """Bytes of one paged block (16 tokens, all KV heads of a layer)."""
        return self.num_kv_heads * 2 * BLOCK_TOKENS * self.head_dim * 2

    @property
    def kv_bytes_per_token(self) -> int:
        return self.block_bytes // BLOCK_TOKENS


TOY = ModelShape(4, 8, 2)                 # BASELINE config 1
LLAMA31_8B = ModelShape(32, 32, 8)        # configs 2, 3, 5
LLAMA31_70B = ModelShape(80, 64, 8)       # config 4 (divide heads by TP)


@dataclass
class _RequestSlabs:
    capacity: int                                     # blocks reserved per slab
    dev: list = field(default_factory=list)           # per layer: pool block or None
    host: list = field(default_factory=list)          # per layer: arena block or None
    staging: list = field(default_factory=list)       # staging slot extents (pool blocks)


class B200Executor:
    """Owns the HBM pool, the pinned host arena, staging and the step runtime."""

    def __init__(self, shape: ModelShape, *, device_blocks: int, host_blocks: int,
                 staging_slots: int = 1, copy_streams: int = 16, seed: int = 0,
                 device: str | torch.device = "cuda", record_timing: bool = False,
                 fill: str = "random", prefetch_next: bool = True, binding: str = "ctypes"):
        if not torch.cuda.is_available():
            raise RuntimeError("B200Executor needs a CUDA device (there is no CPU fallback)")
        if staging_slots not in (1, 2):
            raise ValueError("staging_slots must be 1 (reference rule) or 2 (double buffer)")
        _native.load()
        self.shape = shape
        self.device = torch.device(device)
        self.pool = DevicePool(device_blocks, shape.num_kv_heads, self.device)
        self.host = HostArena(host_blocks, shape.block_bytes)
        self.runtime = StepRuntime(copy_streams, binding=binding)
        self.staging_slots = staging_slots
        self.seed = seed
        self.fill = fill
        self.record_timing = record_timing
        # cross-step prefetch: each step also enqueues the next step's first
        # fetches (same plan, one more token), adopted if the plan is unchanged
        self.prefetch_next = prefetch_next
        self.slabs: dict[int, _RequestSlabs] = {}
        self.layout_version = 0
        self._cached_layout = None
        self.steps = 0
        self.last_timing: dict | None = None
        self.last_inputs: dict | None = None
        self.last_output: torch.Tensor | None = None
        self.migrated = {"h2d_bytes": 0, "d2h_bytes": 0, "moves": 0}
        self.prefill_wall_ms = 0.0
        self._ws = None
        self._mig_start = None        # event before the last un-stepped migration
        self._deferred: list = []     # evicted extents awaiting their D2H
        self._inflight: deque = deque()   # (done event, resources) of un-synced steps
        self._pin_ring: list = []         # pinned [positions | lens] staging per in-flight step
        self._step_dev = None             # device [positions | lens]

    # ------------------------------------------------------------ sizing
    @classmethod
    def for_trace(cls, trace, profile, shape: ModelShape | None = None, max_batch: int = 4,
                  staging_slots: int = 1, **kw) -> "B200Executor":
        """Pools sized for replaying ``trace`` under ``profile`` (engine runs)."""
        if shape is None:
            shape = ModelShape(profile.num_layers, 8, 2)
        caps = [blocks_for_tokens(r.prompt_tokens + r.output_tokens, profile.block_size) + 1
                for r in trace.requests] or [1]
        cap = max(caps)
        per_request = shape.num_layers * cap
        device_blocks = profile.gpu_block_budget + max_batch * per_request // 2 \
            + max_batch * staging_slots * cap + 64
        # the engine keeps batch + paused <= max_batch (src/engine.py:478-504) and a
        # restored layer's host slab is freed, so max_batch * per_request covers
        # every host-resident slab; the factor 2 covers slabs deferred under an
        # in-flight eviction
        host_blocks = 2 * max_batch * per_request + 64
        return cls(shape, device_blocks=device_blocks, host_blocks=host_blocks,
                   staging_slots=staging_slots, **kw)

    # ------------------------------------------------------------ prefill (K5)
    def _prefill(self, rid: int, tokens: int, dsts: list[int]) -> None:
        """Write a fresh request's prompt KV straight to its planned slabs (K5).

        The prompt K/V a prefill would produce (token-major, per layer) is
        synthetic here (seeded N(0,1)); ``dsts[l]`` is the HBM extent or the
        mapped host slab of layer l, so offloaded layers never touch HBM.
        """
        if tokens <= 0:
            return
        from . import ops

        t0 = time.perf_counter()

        hkv = self.shape.num_kv_heads
        per_layer = tokens * hkv * HEAD_DIM * 2 * 2      # K + V bytes of one layer
        chunk = max(1, (1 << 30) // per_layer)
        for lo in range(0, len(dsts), chunk):
            hi = min(len(dsts), lo + chunk)
            shape = (hi - lo, tokens, hkv, HEAD_DIM)
            if self.fill == "zeros":
                k = torch.zeros(shape, dtype=torch.bfloat16, device=self.device)
                v = torch.zeros(shape, dtype=torch.bfloat16, device=self.device)
            else:
                g = torch.Generator(device=self.device)
                g.manual_seed((self.seed * 1_000_003 + rid) * 4099 + lo)
                k = torch.randn(shape, generator=g, device=self.device).to(torch.bfloat16)
                v = torch.randn(shape, generator=g, device=self.device).to(torch.bfloat16)
            dst = torch.tensor(dsts[lo:hi], dtype=torch.int64).to(self.device)
            ops.kv_prefill(k, v, dst)
        # host time of the prefill KV write: a live-wall engine clock excludes it
        # (the reference already charges prefill, src/engine.py:495-503)
        torch.cuda.current_stream().synchronize()
        self.prefill_wall_ms += (time.perf_counter() - t0) * 1e3

    # ------------------------------------------------------------ HBM extents
    def _reclaim(self, wait: bool) -> None:
        """Recycle extents freed under an in-flight eviction once its D2H landed.

        Evicted HBM extents (the D2H source) and host slabs of a request released
        while an eviction may still be writing into them wait here; everything
        else is stream-ordered after the restores (the compute stream waits for
        them, and copy / migration streams start from the compute stream)."""
        if self._deferred and not self.runtime.migration_pending(wait=wait):
            for alloc, start, cap in self._deferred:
                alloc.release(start, cap)
            self._deferred.clear()

    def _free(self, alloc, start: int, cap: int) -> None:
        if self.runtime.migration_pending(wait=False):
            self._deferred.append((alloc, start, cap))
        else:
            alloc.release(start, cap)

    def _alloc(self, alloc, n: int) -> int:
        from .kvpool import PoolExhausted

        self._reclaim(wait=False)
        try:
            return alloc.alloc(n)
        except PoolExhausted:
            if not self._deferred:
                raise
            self._reclaim(wait=True)
            return alloc.alloc(n)

    def _alloc_dev(self, n: int) -> int:
        return self._alloc(self.pool.alloc, n)

    def _alloc_host(self, n: int) -> int:
        return self._alloc(self.host.alloc, n)

    # ------------------------------------------------------------ table sync (K4)
    def _ensure(self, req: RequestState) -> _RequestSlabs:
        st = self.slabs.get(req.id)
        if st is None:
            cap = blocks_for_tokens(req.prompt_tokens + req.target_output_tokens + 1, BLOCK_TOKENS)
            L = self.shape.num_layers
            st = _RequestSlabs(cap, [None] * L, [None] * L, [])
            self.slabs[req.id] = st
        return st

    def _table_differs(self, table, reqs) -> bool:
        """True if making residency equal ``table.locations`` moves anything."""
        if any(rid not in table.locations for rid in self.slabs):
            return True
        for rid, locs in table.locations.items():
            if rid not in reqs:
                continue
            st = self.slabs.get(rid)
            if st is None:
                return True
            if any((loc in _DEVICE_LOCS) != (st.dev[l] is not None) for l, loc in enumerate(locs)):
                return True
        return False

    def sync_table(self, table, batch, paused=()) -> None:
        """Migrate slabs so physical residency equals ``table.locations``.

        The engine re-installs its plan at every step boundary (src/engine.py:
        708-713); when nothing moves this is a no-op, so the layout (and the
        cross-step prefetch the previous step issued) stays valid."""
        reqs = {r.id: r for r in [*batch, *paused]}
        if not self._table_differs(table, reqs):
            return
        # no staging slot or host slab may be reused under an in-flight prefetch
        self.runtime.prefetch_fence()
        for rid in [r for r in self.slabs if r not in table.locations]:
            self.release(rid)
        moves, evicted, restored = [], [], []
        for rid, locs in table.locations.items():
            req = reqs.get(rid)
            if req is None:
                continue
            fresh = rid not in self.slabs
            st = self._ensure(req)
            if fresh:
                # prefill KV goes straight to its placed location
                dsts = []
                for layer, loc in enumerate(locs):
                    if loc in _DEVICE_LOCS:
                        st.dev[layer] = self._alloc_dev(st.capacity)
                        dsts.append(self.pool.addr(st.dev[layer]))
                    else:
                        st.host[layer] = self._alloc_host(st.capacity)
                        dsts.append(self.host.addr(st.host[layer]))
                self._prefill(rid, req.total_tokens, dsts)
                continue
            used = blocks_for_tokens(req.total_tokens, BLOCK_TOKENS)
            nbytes = used * self.shape.block_bytes
            for layer, loc in enumerate(locs):
                on_dev = st.dev[layer] is not None
                if loc in _DEVICE_LOCS and not on_dev:       # restore (H2D)
                    start = self._alloc_dev(st.capacity)
                    st.dev[layer] = start
                    moves.append((self.pool.addr(start), self.host.addr(st.host[layer]), nbytes, 0))
                    # the host copy is dead once restored: later users of that range
                    # (K5 on the compute stream, evictions, fetches) start after the
                    # compute stream's wait for this restore
                    restored.append((st.host[layer], st.capacity))
                    st.host[layer] = None
                elif loc not in _DEVICE_LOCS and on_dev:     # evict (D2H)
                    if st.host[layer] is None:
                        st.host[layer] = self._alloc_host(st.capacity)
                    moves.append((self.host.addr(st.host[layer]), self.pool.addr(st.dev[layer]),
                                  nbytes, 1))
                    evicted.append((self.pool.alloc, st.dev[layer], st.capacity))
                    st.dev[layer] = None
        if moves:
            if self._mig_start is None:
                self._mig_start = torch.cuda.Event(enable_timing=True)
                self._mig_start.record(torch.cuda.current_stream())
            arr = np.array(moves, dtype=np.uint64)
            self.runtime.migrate(arr[:, 0], arr[:, 1], arr[:, 2].astype(np.int64),
                                 arr[:, 3].astype(np.int32), record_timing=self.record_timing)
            for _d, _s, n, kind in moves:
                self.migrated["h2d_bytes" if kind == 0 else "d2h_bytes"] += int(n)
            self.migrated["moves"] += len(moves)
        # Evicted extents are recycled only once their D2H has landed (the
        # eviction overlaps the next step; see ofb_runtime_migrate).
        self._deferred.extend(evicted)
        # Restored layers' host copies are dead; released only now, after the
        # batch is issued, so nothing in this sync reuses a range a restore reads.
        for start, cap in restored:
            self.host.alloc.release(start, cap)
        self.layout_version += 1

    def install(self, batch: list[RequestState], placement: PlacementMatrix) -> None:
        """Make residency equal a placement directly (no engine / BlockTable)."""

        class _Table:
            locations = {rid: ["g" if bit else "h" for bit in row]
                         for rid, row in zip(placement.request_ids, placement.rows)}

        self.sync_table(_Table, batch)

    def release(self, rid: int) -> None:
        st = self.slabs.pop(rid, None)
        if st is None:
            return
        self.runtime.prefetch_fence()
        for start in st.dev:
            if start is not None:
                self.pool.alloc.release(start, st.capacity)
        for start in st.host:      # an eviction may still be writing into these
            if start is not None:
                self._free(self.host.alloc, start, st.capacity)
        for start in st.staging:
            self.pool.alloc.release(start, st.capacity)
        self.layout_version += 1

    # ------------------------------------------------------------ step (K1-K3)
    def _layout(self, batch: list[RequestState]):
        key = (self.layout_version, tuple(r.id for r in batch))
        if self._cached_layout is not None and self._cached_layout[0] == key:
            return self._cached_layout[1]
        L, B = self.shape.num_layers, len(batch)
        width = max(self.slabs[r.id].capacity for r in batch)
        tables = np.full((L, B, width), -1, dtype=np.int32)
        host_slabs = np.zeros((L, B), dtype=np.uint64)
        staging = np.zeros((L, B), dtype=np.uint64)
        for b, req in enumerate(batch):
            st = self.slabs[req.id]
            ramp = np.arange(st.capacity, dtype=np.int32)
            offloaded = [l for l in range(L) if st.dev[l] is None]
            if offloaded and len(st.staging) < self.staging_slots:
                while len(st.staging) < self.staging_slots:
                    st.staging.append(self._alloc_dev(st.capacity))
            for l in range(L):
                if st.dev[l] is not None:
                    tables[l, b, : st.capacity] = st.dev[l] + ramp
            for k, l in enumerate(offloaded):
                slot = st.staging[k % self.staging_slots]
                tables[l, b, : st.capacity] = slot + ramp
                host_slabs[l, b] = self.host.addr(st.host[l])
                staging[l, b] = self.pool.addr(slot)
        layout = {
            "tables": torch.from_numpy(tables).to(self.device),
            "host_dev": torch.from_numpy(host_slabs.view(np.int64)).to(self.device),
            "host": host_slabs, "staging": staging, "width": width,
        }
        self._cached_layout = (key, layout)
        return layout

    def _workspace(self, B: int, max_seq: int) -> torch.Tensor:
        lib = _native.load()
        need = int(lib.ofb_attention_workspace_bytes(B, self.shape.num_q_heads,
                                                     self.shape.num_kv_heads, max_seq))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.zeros(max(need, 1 << 20), dtype=torch.uint8, device=self.device)
        return self._ws

    def synthetic_inputs(self, B: int, step: int | None = None) -> dict:
        """Seeded q / k_new / v_new for one step: bf16 [L, B, H, 128]."""
        g = torch.Generator(device=self.device)
        g.manual_seed(self.seed * 7919 + (self.steps if step is None else step) + 1)
        L, hq, hkv = self.shape.num_layers, self.shape.num_q_heads, self.shape.num_kv_heads
        mk = lambda h: torch.randn((L, B, h, HEAD_DIM), generator=g, device=self.device,  # noqa: E731
                                   dtype=torch.bfloat16)
        return {"q": mk(hq), "k_new": mk(hkv), "v_new": mk(hkv)}

    def prepare_step(self, batch: list[RequestState], inputs: dict | None = None):
        """Build the native step descriptor (no GPU work is enqueued)."""
        for req in batch:
            if req.id not in self.slabs:
                raise RuntimeError(f"request {req.id} has no slabs: install/sync first")
        L, B = self.shape.num_layers, len(batch)
        layout = self._layout(batch)
        positions = np.array([r.total_tokens for r in batch], dtype=np.int32)
        for r, p in zip(batch, positions):
            if p // BLOCK_TOKENS >= self.slabs[r.id].capacity:
                raise RuntimeError(f"request {r.id} outgrew its slab reservation")
        lens = positions + 1
        max_seq = int(lens.max())
        fetch = np.array([blocks_for_tokens(int(p), BLOCK_TOKENS) * self.shape.block_bytes
                          for p in positions], dtype=np.int64)
        if inputs is None:
            inputs = self.synthetic_inputs(B)
        # the attention output: the caller's buffer (a decoder that keeps its
        # descriptors across steps) or a fresh one
        out = inputs["out"] if inputs.get("out") is not None else torch.empty_like(inputs["q"])
        # per-step scalars: pinned ring slot -> one async H2D into a device buffer
        # (stream-ordered, so the previous step has consumed it)
        slot = self.steps % 4
        if len(self._pin_ring) < 4 or self._pin_ring[slot].numel() < 2 * B:
            self._pin_ring = [torch.empty(2 * max(B, 64), dtype=torch.int32).pin_memory()
                              for _ in range(4)]
            self._step_dev = torch.empty(2 * max(B, 64), dtype=torch.int32, device=self.device)
        pin = self._pin_ring[slot]
        pin_np = pin.numpy()
        pin_np[:B] = positions
        pin_np[B:2 * B] = lens
        step_dev = self._step_dev[: 2 * B]
        step_dev.copy_(pin[: 2 * B], non_blocking=True)
        pos_dev, lens_dev = step_dev[:B], step_dev[B:]
        ws = self._workspace(B, max_seq)
        d = _native.StepDesc()
        d.num_layers, d.batch = L, B
        d.num_q_heads, d.num_kv_heads, d.head_dim = (self.shape.num_q_heads,
                                                     self.shape.num_kv_heads, HEAD_DIM)
        d.scale = 1.0 / math.sqrt(HEAD_DIM)
        d.q, d.out = inputs["q"].data_ptr(), out.data_ptr()
        d.k_new, d.v_new = inputs["k_new"].data_ptr(), inputs["v_new"].data_ptr()
        d.kv_pool, d.pool_blocks = self.pool.base, self.pool.blocks
        d.block_tables, d.max_blocks = layout["tables"].data_ptr(), layout["width"]
        d.seq_lens, d.positions = lens_dev.data_ptr(), pos_dev.data_ptr()
        d.host_slabs_dev = layout["host_dev"].data_ptr()
        d.workspace, d.workspace_bytes = ws.data_ptr(), ws.numel()
        d.max_seq_len = max_seq
        d.host_slabs = layout["host"].ctypes.data
        d.staging_dst = layout["staging"].ctypes.data
        d.fetch_bytes = fetch.ctypes.data
        d.staging_slots = self.staging_slots
        d.record_timing = int(self.record_timing)
        next_fetch = None
        if self.prefetch_next:
            next_fetch = np.array([blocks_for_tokens(int(p) + 1, BLOCK_TOKENS) * self.shape.block_bytes
                                   for p in positions], dtype=np.int64)
            d.next_fetch_bytes = next_fetch.ctypes.data
        keep = (inputs, out, pos_dev, lens_dev, ws, layout, fetch, next_fetch)
        return d, keep

    def decode_step(self, batch: list[RequestState], placement: PlacementMatrix | None = None,
                    inputs: dict | None = None, sync: bool = True) -> float | None:
        """Run one decode step on the GPU.

        ``sync=True`` waits for it and returns its device time in ms (the engine
        seam).  ``sync=False`` only enqueues (up to 4 steps in flight) so the host
        prepares the next step while the GPU runs this one; call ``drain()``.
        """
        if placement is not None:
            for req, row in zip(batch, placement.rows):
                st = self.slabs.get(req.id)
                if st is None or any((st.dev[l] is not None) != bool(bit) for l, bit in enumerate(row)):
                    raise RuntimeError("physical residency does not match the placement")
        desc, keep = self.prepare_step(batch, inputs)
        stream = torch.cuda.current_stream()
        t1 = torch.cuda.Event(enable_timing=True)
        if self._mig_start is not None:   # the step also waits for its plan's migration
            t0, self._mig_start = self._mig_start, None
        else:
            t0 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
        self.runtime.decode_step(desc, stream, out=keep[1])
        t1.record(stream)
        self.steps += 1
        self.last_inputs, self.last_output = keep[0], keep[1]
        self.last_positions = np.array([r.total_tokens for r in batch], dtype=np.int32)
        self._inflight.append((t1, keep))
        if not sync:
            while len(self._inflight) > 3:
                self._inflight.popleft()[0].synchronize()
            return None
        t1.synchronize()
        self._inflight.clear()
        if self.record_timing:
            self.last_timing = self.runtime.timing()
        return t0.elapsed_time(t1)

    def drain(self) -> None:
        """Wait for every enqueued step."""
        while self._inflight:
            self._inflight.popleft()[0].synchronize()

    # ------------------------------------------------------------ inspection
    def slab_bits(self, rid: int, layer: int, blocks: int) -> np.ndarray:
        """uint16 [blocks, Hkv, 2, 16, 128] copy of a slab wherever it lives."""
        st = self.slabs[rid]
        shape = (blocks, self.shape.num_kv_heads, 2, BLOCK_TOKENS, HEAD_DIM)
        torch.cuda.synchronize()
        if st.dev[layer] is not None:
            t = self.pool.tensor[st.dev[layer]: st.dev[layer] + blocks]
            return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16).reshape(shape)
        return self.host.view_u16(st.host[layer], blocks).reshape(shape).copy()

    def residency(self, rid: int) -> list[str]:
        st = self.slabs[rid]
        return ["dev" if d is not None else "host" for d in st.dev]

    def close(self) -> None:
        torch.cuda.synchronize()
        self.runtime.close()
        self.host.close()
