"""C1 on B200: the tensor-parallel o-projection fused with its all-reduce (K6).

SURVEY.md 8(e): a KV-head-sharded rank ends each layer's attention with
``attn[B, Hq/N, 128]`` for its own heads; the decoder needs
``hidden[B, H] = sum_r attn_r @ W_o[rows of r]``.  The paper runs NCCL after
the projection.  Here one sm_100a kernel
(``csrc/oproj_allreduce.cu``) computes this rank's partial on the tcgen05
tensor cores and pushes every finished tile straight into each peer's inbox
over NVLink (CUDA-IPC-mapped symmetric buffers), so the exchange overlaps the
math tile by tile; every rank sums the world's tiles in rank order and holds
bit-identical results.

``SymmetricBuffers`` owns this rank's buffer and maps the peers' (handles are
exchanged once with ``torch.distributed.all_gather_object``, any backend).
``SymmetricBuffers.emulated`` gives N ranks inside one process on one GPU -
the only multi-rank configuration a single-GPU box can run - with the kernel
and protocol unchanged (peer pointers are simply local).
"""

from __future__ import annotations

import ctypes

import torch

from . import _native

MAX_WORLD = 8


def _lib():
    return _native.load()


def _check(rc: int, what: str) -> None:
    _native.check(rc, what)


class SymmetricBuffers:
    """One rank's IPC-shareable inbox/flags buffer plus every peer's, mapped here."""

    def __init__(self, world: int, rank: int, max_batch: int, hidden: int, *, group=None,
                 device=None, _peers=None, _owned=True):
        if not 1 <= world <= MAX_WORLD:
            raise ValueError(f"world must be 1..{MAX_WORLD}")
        if not 0 <= rank < world:
            raise ValueError("rank out of range")
        if hidden % 128 or not 1 <= max_batch <= 256:
            raise ValueError("hidden must be a multiple of 128 and 1 <= max_batch <= 256")
        self.world, self.rank = world, rank
        self.max_batch, self.hidden = max_batch, hidden
        self.device = torch.device(device if device is not None else torch.cuda.current_device())
        self.epoch = 0
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._opened: list[int] = []
        self._owned = _owned
        self._group = group
        lib = _lib()
        self._emulated = _peers is not None
        if _peers is not None:           # emulated group: pointers supplied by the factory
            self.ptrs = list(_peers)
            self.local = self.ptrs[rank]
            return
        nbytes = int(lib.ofb_oproj_symm_bytes(world, max_batch, hidden))
        if nbytes <= 0:
            raise ValueError("bad symmetric-buffer geometry")
        with torch.cuda.device(self.device):
            p = ctypes.c_void_p()
            _check(lib.ofb_symm_alloc(nbytes, ctypes.byref(p)), "ofb_symm_alloc")
            self.local = p.value
            self.ptrs = [None] * world
            self.ptrs[rank] = self.local
            if world > 1:
                import torch.distributed as dist

                handle = (ctypes.c_char * 64)()
                _check(lib.ofb_ipc_get_handle(self.local, handle), "ofb_ipc_get_handle")
                gathered = [None] * world
                dist.all_gather_object(gathered, bytes(handle), group=group)
                for r, h in enumerate(gathered):
                    if r == rank:
                        continue
                    buf = (ctypes.c_char * 64).from_buffer_copy(h)
                    q = ctypes.c_void_p()
                    _check(lib.ofb_ipc_open_handle(buf, ctypes.byref(q)), f"ofb_ipc_open_handle(rank {r})")
                    self.ptrs[r] = q.value
                    self._opened.append(q.value)

    @classmethod
    def emulated(cls, world: int, max_batch: int, hidden: int, device=None) -> list["SymmetricBuffers"]:
        """N ranks in this process on one GPU (tests / single-GPU boxes)."""
        lib = _lib()
        nbytes = int(lib.ofb_oproj_symm_bytes(world, max_batch, hidden))
        dev = torch.device(device if device is not None else torch.cuda.current_device())
        ptrs = []
        with torch.cuda.device(dev):
            for _ in range(world):
                p = ctypes.c_void_p()
                _check(lib.ofb_symm_alloc(nbytes, ctypes.byref(p)), "ofb_symm_alloc")
                ptrs.append(p.value)
        return [cls(world, r, max_batch, hidden, device=dev, _peers=ptrs, _owned=(r == 0))
                for r in range(world)]

    def next_epoch(self) -> int:
        # 1..0xFFFFFFFE: parity keeps alternating across the wrap (the inbox /
        # flag slot is epoch & 1)
        self.epoch = (self.epoch % 0xFFFFFFFE) + 1
        return self.epoch

    def check(self) -> None:
        """Raise if any exchange timed out waiting for a peer (synchronises)."""
        if int(self.status.item()) != 0:
            raise RuntimeError(f"rank {self.rank}: a peer's tile never arrived (C1 exchange timed out)")

    def close(self) -> None:
        """Collective when world > 1: no rank frees its buffer while a peer may
        still be writing into it."""
        lib = _lib()
        torch.cuda.synchronize(self.device)
        if self._opened:
            import torch.distributed as dist

            dist.barrier(group=self._group)
        for p in self._opened:
            lib.ofb_ipc_close_handle(p)
        self._opened.clear()
        for p in self._freed_on_close():
            lib.ofb_symm_free(p)
        self.ptrs = []
        self._owned = False

    def _freed_on_close(self) -> list:
        if not self._owned:
            return []
        if self._emulated:          # rank 0 of an emulated group owns every buffer
            return [p for p in self.ptrs if p]
        return [self.local]


def pack_weight(w: torch.Tensor) -> torch.Tensor:
    """[..., H, K] (nn.Linear layout) -> [..., H/128, K/64, 128, 64]: every 128 x 64
    tile K6's TMA loads is 16 KiB contiguous."""
    *lead, h, k = w.shape
    return (w.reshape(*lead, h // 128, 128, k // 64, 64).transpose(-3, -2).contiguous())


def interleave_gate_up(w: torch.Tensor) -> torch.Tensor:
    """[..., 2*I, K] (gate rows, then up rows) -> rows interleaved per 64 (gate
    64t..64t+63, up 64t..64t+63, ...): each 128-row K6 tile then holds matching
    gate and up columns, so its epilogue can emit silu(gate) * up (``swiglu``)."""
    *lead, two_i, k = w.shape
    i = two_i // 2
    if two_i % 2 or i % 64:
        raise ValueError("the gate/up rows must be 2 x a multiple of 64")
    return w.reshape(*lead, 2, i // 64, 64, k).transpose(-4, -3).reshape(*lead, two_i, k)


def deinterleave_gate_up(w: torch.Tensor) -> torch.Tensor:
    """Inverse of ``interleave_gate_up``."""
    *lead, two_i, k = w.shape
    i = two_i // 2
    return w.reshape(*lead, i // 64, 2, 64, k).transpose(-4, -3).reshape(*lead, two_i, k)


class OprojAllReduce:
    """K6: ``hidden[B, H] = sum over ranks of x_r[B, K] @ W_r[H, K]^T`` per layer.

    ``w_o``: bf16 [L, H, K] - the o-projection rows of this rank's heads in
    ``nn.Linear`` layout (K = local q heads x 128).  ``symm=None`` is a single
    rank (the projection alone, no exchange).
    """

    def __init__(self, w_o: torch.Tensor, max_batch: int, symm: SymmetricBuffers | None = None,
                 timeout_ns: int = 0, pack: bool = True):
        if not w_o.is_cuda or w_o.dtype != torch.bfloat16 or w_o.dim() not in (3, 5):
            raise ValueError("w_o must be a bf16 CUDA tensor [layers, hidden, k] "
                             "(or already packed: [layers, hidden/128, k/64, 128, 64])")
        if w_o.dim() == 5:      # packed by the caller (see pack_weight)
            if tuple(w_o.shape[3:]) != (128, 64) or not w_o.is_contiguous():
                raise ValueError("a packed w_o must be contiguous [layers, hidden/128, k/64, 128, 64]")
            self.layers, tiles, chunks = w_o.shape[:3]
            self.hidden, self.k = tiles * 128, chunks * 64
            self.w_layout, self.w = 1, w_o
        else:
            self.layers, self.hidden, self.k = w_o.shape
            if self.k % 64 or self.hidden % 128:
                raise ValueError("k must be a multiple of 64 and hidden of 128")
            # Weights are static: pack once so that every TMA box the kernel loads
            # (128 rows x 64 k of one hidden tile) is 16 KiB contiguous in HBM.
            self.w_layout = 1 if pack else 0
            self.w = pack_weight(w_o) if pack else w_o.contiguous()
        if symm is not None and (symm.hidden != self.hidden or symm.max_batch < max_batch):
            raise ValueError("symmetric buffers sized for another hidden / batch")
        self.max_batch = max_batch
        self.symm = symm
        self.timeout_ns = int(timeout_ns)   # per tile wait; 0 = the library default (5 s)
        lib = _lib()
        nbytes = int(lib.ofb_oproj_workspace_bytes(max_batch, self.k, self.hidden))
        self.ws = torch.zeros(nbytes, dtype=torch.uint8, device=self.w.device)
        self._status = symm.status if symm is not None else torch.zeros(1, dtype=torch.int32,
                                                                         device=self.w.device)

    def __call__(self, x: torch.Tensor, layer: int, out: torch.Tensor | None = None,
                 stream=None, residual: torch.Tensor | None = None,
                 parts: list | None = None, ss_out: torch.Tensor | None = None,
                 ss_in: torch.Tensor | None = None, eps: float = 1e-5,
                 swiglu: bool = False, kv_append: dict | None = None) -> torch.Tensor:
        """Validate, build the descriptor and launch (``prepare`` + ``launch``)."""
        d, result = self.prepare(x, layer, out=out, residual=residual, parts=parts, ss_out=ss_out,
                                 ss_in=ss_in, eps=eps, swiglu=swiglu, kv_append=kv_append)
        s = stream if stream is not None else torch.cuda.current_stream(x.device)
        self.launch(d, s.cuda_stream)
        return result

    def launch(self, d, stream_handle: int) -> None:
        """Launch a descriptor from ``prepare`` (reusable across calls: its tensors
        must stay alive; an exchange takes the next epoch here)."""
        if d.world > 1:
            d.epoch = self.symm.next_epoch()
        _check(_lib().ofb_oproj_allreduce(ctypes.byref(d), ctypes.c_void_p(stream_handle)),
               "ofb_oproj_allreduce")

    def prepare(self, x: torch.Tensor, layer: int, out: torch.Tensor | None = None,
                residual: torch.Tensor | None = None, parts: list | None = None,
                ss_out: torch.Tensor | None = None, ss_in: torch.Tensor | None = None,
                eps: float = 1e-5, swiglu: bool = False, kv_append: dict | None = None):
        """Validate the arguments and build the ``ofb_oproj_desc`` (no launch);
        returns ``(desc, out or parts)``.  ``x``: bf16 [L, B, K] (or [L, B, Hq_local, 128]) - all layers' attention
        output; layer ``layer`` is projected.  A 2-D ``x`` [B, K] is one input for
        every layer (the decoder's residual stream).  Returns bf16 [B, H].
        ``residual`` (bf16 [B, H], may be ``out`` itself) is added before the one
        rounding: the decoder's ``x += o_proj(attn)`` in the same kernel.

        Fused RMSNorm (the whole-decoder step): ``ss_out`` (fp32 [H/128, max_batch])
        receives each hidden tile's per-row sum of squares of the final output;
        ``ss_in`` (such a tensor from the launch that produced ``x``) scales output
        row b by rsqrt(mean(x[b]^2) + eps), so the projection consumes
        RMSNorm(x) with the norm weight folded into W.  ``swiglu``: W was packed
        with ``interleave_gate_up`` and ``out`` is bf16 [B, H/2] = silu(gate) * up.
        ``kv_append`` (with ``parts`` = q, k, v): K3 folded in - the k / v rows are
        also written to the token's slot of the paged pool; keys ``pool``,
        ``tables`` (this layer's [B, max_blocks] int32 device pointer),
        ``positions``, ``host_slabs`` (device pointer or 0), ``max_blocks``,
        ``part`` (index of the k part) and ``block_bytes``."""
        if not x.is_cuda or x.dtype != torch.bfloat16:
            raise ValueError("x must be a bf16 CUDA tensor (no CPU fallback)")
        if x.dim() == 2:             # one input for every layer (W of `layer`)
            x, n_layers = x.reshape(1, *x.shape), 1
        else:
            n_layers = self.layers
            if x.shape[0] != self.layers:
                raise ValueError("x must hold every layer: [layers, batch, ...] (or be [batch, k])")
        b = x.shape[1]
        x = x.reshape(n_layers, b, -1)
        if x.shape[2] != self.k or not x.is_contiguous():
            raise ValueError(f"x must be contiguous [layers, batch, {self.k}]")
        if not 0 <= layer < self.layers:
            raise ValueError("layer out of range")
        w_layer = layer
        if parts is not None:     # column ranges into separate [B, cols] tensors (world 1)
            if out is not None or residual is not None or not 2 <= len(parts) <= 4:
                raise ValueError("parts excludes out / residual and takes 2-4 tensors")
            if self.symm is not None and self.symm.world > 1:
                raise ValueError("parts is a single-rank projection (column-parallel)")
            if sum(t.shape[-1] for t in parts) != self.hidden:
                raise ValueError("the parts' columns must add up to hidden")
            for t in parts:
                if (t.dtype != torch.bfloat16 or not t.is_contiguous() or t.device != x.device
                        or t.reshape(b, -1).shape[1] % 128):
                    raise ValueError("parts must be contiguous bf16 [B, cols] tensors, cols % 128 == 0")
        out_cols = self.hidden // 2 if swiglu else self.hidden
        if out is None and parts is None:
            out = torch.empty((b, out_cols), dtype=torch.bfloat16, device=x.device)
        elif out is not None and (out.shape != (b, out_cols) or out.dtype != torch.bfloat16 or not out.is_contiguous()
              or out.device != x.device):
            raise ValueError(f"out must be a contiguous bf16 [{b}, {out_cols}] tensor on {x.device}")
        for name, t, rows in (("ss_out", ss_out, self.hidden // 128), ("ss_in", ss_in, None)):
            if t is not None and (t.dtype != torch.float32 or not t.is_contiguous() or t.device != x.device
                                  or t.dim() != 2 or t.shape[1] != self.max_batch
                                  or (rows is not None and t.shape[0] != rows)):
                raise ValueError(f"{name} must be a contiguous fp32 [tiles, max_batch={self.max_batch}] tensor")
        d = _native.OprojDesc()
        d.x, d.w = x.data_ptr(), self.w.data_ptr()
        d.out = out.data_ptr() if out is not None else None
        if parts is not None:
            d.out_parts = len(parts)
            for i, t in enumerate(parts):
                d.part_cols[i] = t.reshape(b, -1).shape[1]
                d.part_out[i] = t.data_ptr()
        d.layers, d.layer, d.batch, d.k, d.hidden = self.layers, w_layer, b, self.k, self.hidden
        if n_layers == 1 and self.layers > 1:
            # one x for every layer: a per-call map over [1, batch, k], W of layer w_layer
            d.x_layers = 1
        if ss_out is not None:
            d.ss_out = ss_out.data_ptr()
        if ss_in is not None:
            d.ss_in, d.ss_tiles = ss_in.data_ptr(), ss_in.shape[0]
        d.eps = float(eps)
        d.swiglu = 1 if swiglu else 0
        if kv_append is not None:
            if parts is None:
                raise ValueError("kv_append needs the q / k / v parts")
            d.kv_pool, d.kv_tables = kv_append["pool"], kv_append["tables"]
            d.kv_positions, d.kv_host_slabs = kv_append["positions"], kv_append.get("host_slabs") or None
            d.kv_max_blocks, d.kv_part = kv_append["max_blocks"], kv_append["part"]
            d.kv_block_bytes = kv_append["block_bytes"]
        d.workspace, d.workspace_bytes = self.ws.data_ptr(), self.ws.numel()
        d.max_batch = self.max_batch
        d.status = self._status.data_ptr()
        d.timeout_ns = self.timeout_ns
        d.w_layout = self.w_layout
        if residual is not None:
            if (residual.shape != out.shape or residual.dtype != torch.bfloat16
                    or not residual.is_contiguous() or residual.device != x.device):
                raise ValueError(f"residual must be a contiguous bf16 [{b}, {self.hidden}] tensor")
            d.residual = residual.data_ptr()
        if self.symm is None or self.symm.world == 1:
            d.world, d.rank, d.epoch = 1, 0, 1
            if self.symm is not None:
                d.symm[0] = self.symm.local
        else:
            d.world, d.rank = self.symm.world, self.symm.rank
            for r, p in enumerate(self.symm.ptrs):
                d.symm[r] = p
            d.epoch = 1                  # the real epoch is taken at launch
        return d, (out if parts is None else parts)
