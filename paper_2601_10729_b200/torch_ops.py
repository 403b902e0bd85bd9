"""``torch.ops.orbit`` - the data-path ops registered with the torch dispatcher.

SURVEY.md 8(b) names the boundary as extension ops in a ``TORCH_LIBRARY``
namespace: ``orbit::decode_attention`` (K1), ``orbit::kv_append`` (K3),
``orbit::kv_prefill`` (K5), ``orbit::decode_step`` (K3+K2+K1 of a whole step,
through the native runtime) and ``orbit::migrate`` (K4).  They are registered
by ``csrc/torch_ops.cpp`` (``liborbit_torch_ops.so``), a thin C++ layer over the
same C ABI the ctypes binding (``ops.py`` / ``runtime.py``) calls - one set of
kernels, two bindings.  Registered ops can be captured in CUDA graphs through
``torch.ops`` and traced by ``torch.compile``; the fake (meta) kernels below give
their output metadata without touching a GPU.  There is no CPU kernel: a CPU
tensor raises.
"""

from __future__ import annotations

import math
import threading

import torch

from . import _native

_LOCK = threading.Lock()
_LOADED = False


def load() -> None:
    """Load (building first if needed) the registration library; idempotent."""
    global _LOADED
    with _LOCK:
        if _LOADED:
            return
        from . import build as _build

        path = _build.torch_ops_path()
        if not path.exists():
            _build.build_torch_ops()
        _native.load()            # the kernel library first: same file the .so links
        torch.ops.load_library(str(path))
        _register_fakes()
        _LOADED = True


def _register_fakes() -> None:
    lib = "orbit::"

    @torch.library.register_fake(lib + "decode_attention")
    def _(q, kv_pool, block_tables, seq_lens, max_seq_len, scale, ws):
        return torch.empty_like(q)

    @torch.library.register_fake(lib + "kv_append")
    def _(k_new, v_new, kv_pool, block_tables, positions, host_slabs):
        return None

    @torch.library.register_fake(lib + "kv_prefill")
    def _(k, v, dst):
        return None

    @torch.library.register_fake(lib + "decode_step")
    def _(runtime, desc, out):
        return None

    @torch.library.register_fake(lib + "migrate")
    def _(runtime, dst, src, nbytes, kinds, record_timing, stream_of):
        return None


def decode_attention(q, kv_pool, block_tables, seq_lens, max_seq_len: int, *, scale=None,
                     ws=None, out=None):
    """``orbit::decode_attention`` with ops.decode_attention's defaults (scale
    1/sqrt(128), cached workspace)."""
    from . import ops

    load()
    if scale is None:
        scale = 1.0 / math.sqrt(128)
    if ws is None:
        ws = ops.workspace(q.shape[0], q.shape[1], kv_pool.shape[1], max_seq_len, q.device)
    if out is None:
        return torch.ops.orbit.decode_attention(q, kv_pool, block_tables, seq_lens,
                                                int(max_seq_len), float(scale), ws)
    return torch.ops.orbit.decode_attention.out(q, kv_pool, block_tables, seq_lens,
                                                int(max_seq_len), float(scale), ws, out=out)


def kv_append(k_new, v_new, kv_pool, block_tables, positions, host_slabs=None) -> None:
    """``orbit::kv_append``; accepts one layer ([B, Hkv, 128]) like ops.kv_append."""
    load()
    if k_new.dim() == 3:
        k_new, v_new = k_new.unsqueeze(0), v_new.unsqueeze(0)
        if block_tables.dim() == 2:
            block_tables = block_tables.unsqueeze(0)
        if host_slabs is not None and host_slabs.dim() == 1:
            host_slabs = host_slabs.unsqueeze(0)
    torch.ops.orbit.kv_append(k_new.contiguous(), v_new.contiguous(), kv_pool,
                              block_tables.contiguous(), positions, host_slabs)


def kv_prefill(k, v, dst_addrs) -> None:
    load()
    torch.ops.orbit.kv_prefill(k.contiguous(), v.contiguous(), dst_addrs)
