"""Thin Python handle on the native step runtime (``ofb_runtime``).

The runtime owns the copy streams and events; every call only enqueues work
(no host blocking) except ``timing()``, which waits on the recorded events.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class StepRuntime:
    """K2/K4 copy-engine orchestration + K1/K3 launches for whole steps.

    ``binding`` picks how steps and migrations reach the library: ``"ctypes"``
    (the C ABI directly) or ``"torch"`` (the dispatcher ops ``orbit::decode_step``
    / ``orbit::migrate`` registered over the same ABI, ``torch_ops.py``)."""

    def __init__(self, max_copy_streams: int = 16, binding: str = "ctypes"):
        if binding not in ("ctypes", "torch"):
            raise ValueError(f"unknown binding {binding!r}")
        self.binding = binding
        if binding == "torch":
            from . import torch_ops

            torch_ops.load()
        self.lib = _native.load()
        handle = self.lib.ofb_runtime_create(max_copy_streams)
        if not handle:
            raise _native.NativeError(f"ofb_runtime_create: {self.lib.ofb_last_error().decode()}")
        self.handle = handle

    def decode_step(self, desc: _native.StepDesc, stream=None, out: torch.Tensor | None = None) -> None:
        s = stream if stream is not None else torch.cuda.current_stream()
        if self.binding == "torch":
            if out is None:
                raise ValueError("the torch binding needs the step's output tensor")
            with torch.cuda.stream(s):
                torch.ops.orbit.decode_step(int(self.handle), ctypes.addressof(desc), out)
            return
        rc = self.lib.ofb_runtime_decode_step(self.handle, ctypes.byref(desc), s.cuda_stream)
        _native.check(rc, "ofb_runtime_decode_step")

    def step_begin(self, desc: _native.StepDesc, stream=None) -> None:
        s = stream if stream is not None else torch.cuda.current_stream()
        rc = self.lib.ofb_runtime_step_begin(self.handle, ctypes.byref(desc), s.cuda_stream)
        _native.check(rc, "ofb_runtime_step_begin")

    def step_layers(self, count: int) -> None:
        _native.check(self.lib.ofb_runtime_step_layers(self.handle, count), "ofb_runtime_step_layers")

    def step_end(self) -> None:
        _native.check(self.lib.ofb_runtime_step_end(self.handle), "ofb_runtime_step_end")

    def step_abort(self) -> None:
        """Drop a step after a caller-side failure (never raises a second error)."""
        self.lib.ofb_runtime_step_abort(self.handle)

    def prefetch_fence(self, stream=None) -> None:
        s = stream if stream is not None else torch.cuda.current_stream()
        _native.check(self.lib.ofb_runtime_prefetch_fence(self.handle, s.cuda_stream),
                      "ofb_runtime_prefetch_fence")

    def prefetch_stats(self) -> dict:
        a, d = ctypes.c_int64(), ctypes.c_int64()
        _native.check(self.lib.ofb_runtime_prefetch_stats(self.handle, ctypes.byref(a), ctypes.byref(d)),
                      "ofb_runtime_prefetch_stats")
        return {"adopted": a.value, "dropped": d.value}

    def migrate(self, dst: np.ndarray, src: np.ndarray, nbytes: np.ndarray, kinds: np.ndarray,
                record_timing: bool = False, stream=None) -> None:
        n = len(dst)
        if n == 0:
            return
        dst = np.ascontiguousarray(dst, dtype=np.uint64)
        src = np.ascontiguousarray(src, dtype=np.uint64)
        nbytes = np.ascontiguousarray(nbytes, dtype=np.int64)
        kinds = np.ascontiguousarray(kinds, dtype=np.int32)
        s = stream if stream is not None else torch.cuda.current_stream()
        if self.binding == "torch":
            anchor = torch.empty(0, device=s.device)
            with torch.cuda.stream(s):
                torch.ops.orbit.migrate(int(self.handle), torch.from_numpy(dst.view(np.int64)),
                                        torch.from_numpy(src.view(np.int64)),
                                        torch.from_numpy(nbytes), torch.from_numpy(kinds),
                                        bool(record_timing), anchor)
            return
        rc = self.lib.ofb_runtime_migrate(self.handle, n, _ptr(dst), _ptr(src), _ptr(nbytes),
                                          _ptr(kinds), int(record_timing), s.cuda_stream)
        _native.check(rc, "ofb_runtime_migrate")

    def migration_pending(self, wait: bool = False) -> bool:
        rc = self.lib.ofb_runtime_migration_pending(self.handle, int(wait))
        if rc < 0 or rc > 1:
            _native.check(rc, "ofb_runtime_migration_pending")
        return rc == 1

    def timing(self) -> dict:
        t = _native.StepTiming()
        _native.check(self.lib.ofb_runtime_timing(self.handle, ctypes.byref(t)), "ofb_runtime_timing")
        return {name: getattr(t, name) for name, _ in _native.StepTiming._fields_}

    def stream_stats(self) -> list[dict]:
        """Per copy stream: bytes fetched and busy ms over the timed steps."""
        n = 64
        b = (ctypes.c_double * n)()
        t = (ctypes.c_double * n)()
        k = ctypes.c_int32()
        _native.check(self.lib.ofb_runtime_stream_stats(self.handle, n, b, t, ctypes.byref(k)),
                      "ofb_runtime_stream_stats")
        return [{"bytes": b[i], "busy_ms": t[i]} for i in range(min(k.value, n))]

    def timing_reset(self) -> None:
        _native.check(self.lib.ofb_runtime_timing_reset(self.handle), "ofb_runtime_timing_reset")

    def close(self) -> None:
        if self.handle:
            self.lib.ofb_runtime_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def link_probe(host_addr: int, dev_addr: int, nbytes: int, reps: int = 10) -> tuple[float, float]:
    """Best-of-``reps`` pinned H2D / D2H GB/s over ``nbytes``."""
    lib = _native.load()
    h2d = ctypes.c_double()
    d2h = ctypes.c_double()
    _native.check(lib.ofb_link_probe(host_addr, dev_addr, nbytes, reps, ctypes.byref(h2d),
                                     ctypes.byref(d2h)), "ofb_link_probe")
    return h2d.value, d2h.value
