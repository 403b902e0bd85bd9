"""Torch-facing wrappers of the sm_100a ops (K1 attention, K3 append).

Tensors are borrowed for the duration of a call; the library never frees
them.  All ops run on the caller's current CUDA stream and raise on CPU
tensors - there is no CPU fallback on the product path.

KV block layout (pool, staging, host slabs): ``bf16 [blocks][Hkv][2][16][128]``.
"""

from __future__ import annotations

import ctypes
import math

import torch

from . import _native

HEAD_DIM = 128
BLOCK_TOKENS = 16

_WORKSPACES: dict[int, torch.Tensor] = {}


def _stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _need_cuda(*tensors) -> None:
    for t in tensors:
        if t is not None and not t.is_cuda:
            raise ValueError("orbitflow ops run on the GPU only (no CPU fallback); got a CPU tensor")


def workspace(batch: int, hq: int, hkv: int, max_seq_len: int, device) -> torch.Tensor:
    """Zero-initialised scratch for K1, grown on demand and cached per device."""
    lib = _native.load()
    need = int(lib.ofb_attention_workspace_bytes(batch, hq, hkv, max_seq_len))
    dev = torch.device(device)
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    ws = _WORKSPACES.get(key)
    if ws is None or ws.numel() < need:
        ws = torch.zeros(max(need, 1 << 20), dtype=torch.uint8, device=dev)
        _WORKSPACES[key] = ws
    return ws


def decode_attention(q: torch.Tensor, kv_pool: torch.Tensor, block_tables: torch.Tensor,
                     seq_lens: torch.Tensor, *, max_seq_len: int | None = None,
                     scale: float | None = None, out: torch.Tensor | None = None,
                     ws: torch.Tensor | None = None) -> torch.Tensor:
    """GQA decode attention of one layer over paged KV.

    q: bf16 [B, Hq, 128]; kv_pool: bf16 [nblocks, Hkv, 2, 16, 128];
    block_tables: int32 [B, max_blocks]; seq_lens: int32 [B] (device).
    """
    _need_cuda(q, kv_pool, block_tables, seq_lens, out, ws)
    if q.dtype != torch.bfloat16 or kv_pool.dtype != torch.bfloat16:
        raise ValueError("q and kv_pool must be bf16")
    if block_tables.dtype != torch.int32 or seq_lens.dtype != torch.int32:
        raise ValueError("block_tables and seq_lens must be int32")
    batch, hq, d = q.shape
    if d != HEAD_DIM:
        raise ValueError("head_dim must be 128")
    nblocks, hkv = kv_pool.shape[0], kv_pool.shape[1]
    if tuple(kv_pool.shape[2:]) != (2, BLOCK_TOKENS, HEAD_DIM):
        raise ValueError("kv_pool must be [blocks, Hkv, 2, 16, 128]")
    if max_seq_len is None:
        max_seq_len = int(seq_lens.max().item()) if batch else 0
    if scale is None:
        scale = 1.0 / math.sqrt(HEAD_DIM)
    q = q.contiguous()
    block_tables = block_tables.contiguous()
    if out is None:
        out = torch.empty_like(q)
    if ws is None:
        ws = workspace(batch, hq, hkv, max_seq_len, q.device)
    lib = _native.load()
    rc = lib.ofb_decode_attention(
        q.data_ptr(), out.data_ptr(), kv_pool.data_ptr(), nblocks, block_tables.data_ptr(),
        block_tables.shape[1], seq_lens.data_ptr(), ws.data_ptr(), ws.numel(), batch, hq, hkv,
        d, int(max_seq_len), float(scale), _stream_ptr())
    _native.check(rc, "ofb_decode_attention")
    return out


def kv_append(k_new: torch.Tensor, v_new: torch.Tensor, kv_pool: torch.Tensor | None,
              block_tables: torch.Tensor | None, positions: torch.Tensor,
              host_slabs: torch.Tensor | None = None) -> None:
    """Write the new token's K/V rows (all layers in k_new's leading dim).

    k_new/v_new: bf16 [L, B, Hkv, 128] (or [B, Hkv, 128] for one layer);
    block_tables: int32 [L, B, max_blocks] (or [B, max_blocks]);
    positions: int32 [B]; host_slabs: uint64-as-int64 [L, B] mapped host
    slab addresses (0 = none).
    """
    _need_cuda(k_new, v_new, kv_pool, block_tables, positions, host_slabs)
    if k_new.dim() == 3:
        k_new, v_new = k_new.unsqueeze(0), v_new.unsqueeze(0)
        if block_tables is not None and block_tables.dim() == 2:
            block_tables = block_tables.unsqueeze(0)
        if host_slabs is not None and host_slabs.dim() == 1:
            host_slabs = host_slabs.unsqueeze(0)
    layers, batch, hkv, d = k_new.shape
    lib = _native.load()
    rc = lib.ofb_kv_append(
        k_new.contiguous().data_ptr(), v_new.contiguous().data_ptr(),
        kv_pool.data_ptr() if kv_pool is not None else None,
        block_tables.contiguous().data_ptr() if block_tables is not None else None,
        block_tables.shape[-1] if block_tables is not None else 0,
        positions.data_ptr(),
        host_slabs.contiguous().data_ptr() if host_slabs is not None else None,
        layers, batch, hkv, d, _stream_ptr())
    _native.check(rc, "ofb_kv_append")


def device_info() -> tuple[int, int]:
    lib = _native.load()
    sms = _native.c_i32()
    occ = _native.c_i32()
    _native.check(lib.ofb_device_info(ctypes.byref(sms), ctypes.byref(occ)), "ofb_device_info")
    return sms.value, occ.value


def set_attention_kernel(variant: str) -> str:
    """Select K1's work decomposition: "stream" (persistent stream-K), "split"
    (fixed splits + last-CTA combine), "cluster" (cluster splits, DSMEM combine),
    "split2" (fixed splits + a second, programmatically launched combine kernel)
    or "auto" (default).  Returns the previous one."""
    names = {"stream": 0, "split": 1, "auto": 2, "cluster": 3, "split2": 4}
    prev = _native.load().ofb_set_attention_kernel(names[variant])
    if prev < 0:
        _native.check(prev, "ofb_set_attention_kernel")
    return {v: k for k, v in names.items()}[prev]


def cluster_plan(batch: int, hkv: int, max_seq_len: int) -> dict | None:
    """The cluster K1's plan on this GPU (None: not a one-wave cluster shape)."""
    lib = _native.load()
    slots = (ctypes.c_int32 * 5)()
    _native.check(lib.ofb_attention_cluster_slots(slots), "ofb_attention_cluster_slots")
    out = [ctypes.c_int32() for _ in range(4)]
    rc = lib.ofb_attention_cluster_plan(batch, hkv, max_seq_len, slots, *[ctypes.byref(o) for o in out])
    if rc != 0:
        return None
    return {"cluster": out[0].value, "clusters_per_pair": out[1].value,
            "blocks_per_cta": out[2].value, "stages": out[3].value, "slots": list(slots)}


def kv_prefill(k: torch.Tensor, v: torch.Tensor, dst_addrs: torch.Tensor) -> None:
    """K5: scatter prompt K/V (bf16 [L, P, Hkv, 128]) into the paged layout of the
    L slabs at ``dst_addrs`` (int64 device tensor of HBM or mapped-host addresses)."""
    _need_cuda(k, v, dst_addrs)
    layers, tokens, hkv, d = k.shape
    lib = _native.load()
    rc = lib.ofb_kv_prefill(k.contiguous().data_ptr(), v.contiguous().data_ptr(),
                            dst_addrs.data_ptr(), layers, tokens, hkv, d, _stream_ptr())
    _native.check(rc, "ofb_kv_prefill")
