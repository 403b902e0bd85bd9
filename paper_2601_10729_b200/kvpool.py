"""Physical KV memory: the HBM block pool, the pinned host arena, extents.

Layout (SURVEY.md 8(a) note; "1D flattened, layer-aware"):
one paged block = 16 tokens x all KV heads of one layer =
``bf16 [Hkv][2][16][128]`` (Hkv * 8 KiB).  The HBM pool is one flat array of
such blocks; a (request, layer) slab is an *extent* (contiguous run of
blocks, capacity = prompt + target output) addressed through the per-layer
block table the attention kernel reads, so a whole-slab DMA is one copy.
Staging slots for streamed layers are extents of the same pool, so the
kernel reads resident and staged slabs identically.  Host slabs live in one
pinned, device-mapped arena (``ofb_host_alloc``) with the same layout.

Allocation is deterministic first-fit over a sorted free list with
coalescing; there is no reference counterpart (kvsim tracks only locations
and counts, engine.py:126-210), so determinism is the only contract.
"""

from __future__ import annotations

import bisect
import ctypes

import numpy as np
import torch

from . import _native

HEAD_DIM = 128
BLOCK_TOKENS = 16


class PoolExhausted(RuntimeError):
    """No free extent large enough (physical HBM / host capacity)."""


class ExtentAllocator:
    """First-fit allocator of block extents over [0, capacity)."""

    def __init__(self, capacity: int):
        if capacity < 0:
            raise ValueError("capacity must be >= 0")
        self.capacity = capacity
        self._starts: list[int] = [0] if capacity else []
        self._lengths: dict[int, int] = {0: capacity} if capacity else {}
        self.in_use = 0

    def alloc(self, n: int) -> int:
        if n <= 0:
            raise ValueError("extent length must be > 0")
        for start in self._starts:
            length = self._lengths[start]
            if length >= n:
                self._starts.remove(start)
                del self._lengths[start]
                if length > n:
                    self._insert(start + n, length - n)
                self.in_use += n
                return start
        raise PoolExhausted(f"no free extent of {n} blocks ({self.capacity - self.in_use} free, "
                            f"fragmented into {len(self._starts)} runs)")

    def _insert(self, start: int, length: int) -> None:
        bisect.insort(self._starts, start)
        self._lengths[start] = length

    def release(self, start: int, n: int) -> None:
        if n <= 0:
            return
        if start < 0 or start + n > self.capacity:
            raise ValueError("extent outside the pool")
        i = bisect.bisect_left(self._starts, start)
        nxt = self._starts[i] if i < len(self._starts) else None
        prev = self._starts[i - 1] if i > 0 else None
        if (nxt is not None and nxt < start + n) or (
                prev is not None and prev + self._lengths[prev] > start):
            raise ValueError("double free (extent overlaps a free run)")
        self.in_use -= n
        if nxt is not None and nxt == start + n:          # merge with the following run
            self._starts.pop(i)
            n += self._lengths.pop(nxt)
        if prev is not None and prev + self._lengths[prev] == start:   # and the preceding one
            self._lengths[prev] += n
            return
        self._insert(start, n)

    @property
    def free_blocks(self) -> int:
        return self.capacity - self.in_use


class DevicePool:
    """HBM block pool: ``bf16 [blocks, Hkv, 2, 16, 128]`` on one device."""

    def __init__(self, blocks: int, num_kv_heads: int, device):
        self.blocks = blocks
        self.num_kv_heads = num_kv_heads
        self.block_bytes = num_kv_heads * 2 * BLOCK_TOKENS * HEAD_DIM * 2
        self.tensor = torch.empty((blocks, num_kv_heads, 2, BLOCK_TOKENS, HEAD_DIM),
                                  dtype=torch.bfloat16, device=device)
        self.alloc = ExtentAllocator(blocks)

    @property
    def base(self) -> int:
        return self.tensor.data_ptr()

    def addr(self, block: int) -> int:
        return self.base + block * self.block_bytes


class HostArena:
    """Pinned, device-mapped host memory holding host-resident KV slabs."""

    def __init__(self, blocks: int, block_bytes: int):
        self.blocks = blocks
        self.block_bytes = block_bytes
        self.nbytes = max(1, blocks) * block_bytes
        lib = _native.load()
        ptr = lib.ofb_host_alloc(self.nbytes)
        if not ptr:
            raise _native.NativeError(f"pinned host allocation of {self.nbytes} bytes failed: "
                                      f"{lib.ofb_last_error().decode()}")
        self.base = int(ptr)
        self.alloc = ExtentAllocator(blocks)

    def addr(self, block: int) -> int:
        return self.base + block * self.block_bytes

    def view_u16(self, block: int, count: int) -> np.ndarray:
        """numpy uint16 view (bf16 bits) of ``count`` blocks - for checks."""
        nbytes = count * self.block_bytes
        buf = (ctypes.c_uint8 * nbytes).from_address(self.addr(block))
        return np.frombuffer(buf, dtype=np.uint16)

    def close(self) -> None:
        if self.base:
            _native.load().ofb_host_free(self.base)
            self.base = 0

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass
