"""CPU oracle - TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` arm may import this package, and only as the checker or
the timed CPU baseline; the product package never imports it.

Contents (each C function cites the reference file:line it restates):
  * attn_oracle.c      GQA decode attention + append over the paged layout
                       (attention math: parity unpinned by the reference,
                       which has no attention - see the C header)
  * schedule_oracle.c  float transfer schedule, fetch volume, Eq. 1 buffer,
                       reconfiguration delta (kvsim/latency.py)
Build: ``make -C oracle`` -> ``oracle/build/liboracle.so``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "build" / "liboracle.so"
_LIB = None


def build() -> Path:
    srcs = list(HERE.glob("*.c")) + [HERE / "Makefile"]
    if not LIB_PATH.exists() or any(p.stat().st_mtime > LIB_PATH.stat().st_mtime for p in srcs):
        subprocess.run(["make", "-C", str(HERE)], check=True, capture_output=True)
    return LIB_PATH


def lib():
    global _LIB
    if _LIB is None:
        build()
        L = ctypes.CDLL(str(LIB_PATH))
        vp, i32, i64, f32, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_double
        L.oracle_decode_attention.argtypes = [vp, vp, vp, i32, vp, vp, i32, i32, i32, f32, i32]
        L.oracle_decode_attention.restype = None
        L.oracle_kv_append.argtypes = [vp, vp, vp, vp, i32, vp, i32, i32]
        L.oracle_kv_append.restype = None
        L.oracle_stall_schedule.argtypes = [i32, vp, vp, i32, f64, f64, vp]
        L.oracle_stall_schedule.restype = f64
        L.oracle_blocks_to_fetch.argtypes = [i32, vp, vp, i32]
        L.oracle_blocks_to_fetch.restype = i64
        L.oracle_prefetch_buffer.argtypes = [i32, vp, vp, i32]
        L.oracle_prefetch_buffer.restype = i64
        L.oracle_reconfiguration_delta.argtypes = [i32, vp, vp, vp, i32, vp]
        L.oracle_reconfiguration_delta.restype = None
        _LIB = L
    return _LIB


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def host_threads() -> int:
    return len(os.sched_getaffinity(0))


# ---------------------------------------------------------------- attention
def decode_attention(q_bf16: np.ndarray, pool_bf16: np.ndarray, block_tables: np.ndarray,
                     seq_lens: np.ndarray, scale: float, threads: int | None = None) -> np.ndarray:
    """q: uint16 (bf16 bits) [B, Hq, 128]; pool: uint16 [nblk, Hkv, 2, 16, 128];
    block_tables: int32 [B, max_blocks]; seq_lens: int32 [B].  Returns f32 [B, Hq, 128]."""
    q = np.ascontiguousarray(q_bf16, dtype=np.uint16)
    pool = np.ascontiguousarray(pool_bf16, dtype=np.uint16)
    bt = np.ascontiguousarray(block_tables, dtype=np.int32)
    sl = np.ascontiguousarray(seq_lens, dtype=np.int32)
    b, hq, _ = q.shape
    hkv = pool.shape[1]
    out = np.zeros((b, hq, 128), dtype=np.float32)
    lib().oracle_decode_attention(_ptr(q), _ptr(pool), _ptr(bt), bt.shape[1], _ptr(sl), _ptr(out),
                                  b, hq, hkv, scale, threads or host_threads())
    return out


def kv_append(k_new: np.ndarray, v_new: np.ndarray, pool: np.ndarray, block_tables: np.ndarray,
              positions: np.ndarray) -> None:
    """In-place append of one layer into ``pool`` (uint16 bf16 bits)."""
    assert pool.flags.c_contiguous and pool.dtype == np.uint16
    k = np.ascontiguousarray(k_new, dtype=np.uint16)
    v = np.ascontiguousarray(v_new, dtype=np.uint16)
    bt = np.ascontiguousarray(block_tables, dtype=np.int32)
    pos = np.ascontiguousarray(positions, dtype=np.int32)
    lib().oracle_kv_append(_ptr(k), _ptr(v), _ptr(pool), _ptr(bt), bt.shape[1], _ptr(pos),
                           k.shape[0], k.shape[1])


def dense_attention_f64(q: np.ndarray, k: np.ndarray, v: np.ndarray, scale: float) -> np.ndarray:
    """Independent float64 dense reference: q [Hq, d], k/v [T, Hkv, d]."""
    hq = q.shape[0]
    hkv = k.shape[1]
    g = hq // hkv
    out = np.empty((hq, q.shape[1]))
    for h in range(hq):
        kk = k[:, h // g, :].astype(np.float64)
        s = kk @ q[h].astype(np.float64) * scale
        s = np.exp(s - s.max())
        out[h] = (s[:, None] * v[:, h // g, :].astype(np.float64)).sum(0) / s.sum()
    return out


# ---------------------------------------------------------------- schedule
def _sched_inputs(sizes, offloaded):
    s = np.ascontiguousarray(sizes, dtype=np.int64)
    off = np.ascontiguousarray(offloaded, dtype=np.uint8)
    return s, off, off.shape[1] if off.ndim == 2 else 0


def stall_schedule(sizes, offloaded, comp: float, bw: float):
    """(total latency ms, per-layer stalls) - float restatement of _simulate_stalls."""
    s, off, L = _sched_inputs(sizes, offloaded)
    stalls = np.zeros(max(L, 1), dtype=np.float64)
    total = lib().oracle_stall_schedule(len(s), _ptr(s), _ptr(off), L, comp, bw, _ptr(stalls))
    return total, stalls[:L]


def blocks_to_fetch(sizes, offloaded) -> int:
    s, off, L = _sched_inputs(sizes, offloaded)
    return int(lib().oracle_blocks_to_fetch(len(s), _ptr(s), _ptr(off), L))


def prefetch_buffer(sizes, offloaded) -> int:
    s, off, L = _sched_inputs(sizes, offloaded)
    return int(lib().oracle_prefetch_buffer(len(s), _ptr(s), _ptr(off), L))


def reconfiguration_delta(sizes, old_resident, new_resident) -> tuple[int, int]:
    s = np.ascontiguousarray(sizes, dtype=np.int64)
    a = np.ascontiguousarray(old_resident, dtype=np.uint8)
    b = np.ascontiguousarray(new_resident, dtype=np.uint8)
    out = np.zeros(2, dtype=np.int64)
    lib().oracle_reconfiguration_delta(len(s), _ptr(s), _ptr(a), _ptr(b), a.shape[1], _ptr(out))
    return int(out[0]), int(out[1])
