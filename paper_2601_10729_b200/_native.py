"""ctypes binding of the sm_100a C ABI (``include/orbitflow_b200.h``).

The library is the only compute path: if it is missing or fails to load the
ops raise; nothing falls back to a CPU implementation.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

_LOCK = threading.Lock()
_LIB = None

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_f32 = ctypes.c_float
c_f64 = ctypes.c_double
c_vp = ctypes.c_void_p
c_u64p = ctypes.POINTER(ctypes.c_uint64)
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_i32p = ctypes.POINTER(ctypes.c_int32)


class StepDesc(ctypes.Structure):
    """Mirror of ``ofb_step_desc``."""

    _fields_ = [
        ("num_layers", c_i32), ("batch", c_i32), ("num_q_heads", c_i32),
        ("num_kv_heads", c_i32), ("head_dim", c_i32),
        ("scale", c_f32),
        ("q", c_vp), ("out", c_vp), ("k_new", c_vp), ("v_new", c_vp),
        ("kv_pool", c_vp), ("pool_blocks", c_i64),
        ("block_tables", c_vp), ("max_blocks", c_i32),
        ("seq_lens", c_vp), ("positions", c_vp), ("host_slabs_dev", c_vp),
        ("workspace", c_vp), ("workspace_bytes", c_i64),
        ("max_seq_len", c_i32),
        ("host_slabs", c_vp), ("staging_dst", c_vp), ("fetch_bytes", c_vp),
        ("staging_slots", c_i32), ("record_timing", c_i32),
        ("next_fetch_bytes", c_vp),
        ("append_per_layer", c_i32),
    ]


class StepTiming(ctypes.Structure):
    """Mirror of ``ofb_step_timing``."""

    _fields_ = [
        ("layers", c_i32), ("attn_ms_total", c_f32), ("attn_ms_max", c_f32),
        ("copies", c_i32), ("copy_ms_sum", c_f32), ("copy_bytes", c_f64),
        ("copy_span_ms", c_f32), ("step_ms", c_f32), ("copy_streams", c_i32),
        ("mig_ms", c_f32), ("mig_h2d_bytes", c_f64), ("mig_d2h_bytes", c_f64),
        ("acc_steps", c_i32), ("acc_attn_launches", c_i32), ("acc_attn_ms", c_f64),
        ("acc_copy_bytes", c_f64), ("acc_step_ms", c_f64),
    ]


class PlanProblem(ctypes.Structure):
    """Mirror of ``ofb_plan_problem``."""

    _fields_ = [
        ("num_layers", c_i32), ("batch", c_i32), ("num_paused", c_i32), ("block_size", c_i32),
        ("compute_base_ms", c_f64), ("compute_per_token_ms", c_f64),
        ("bandwidth_blocks_per_ms", c_f64), ("gpu_block_budget", c_i64),
        ("tbt_ms", c_f64), ("violation_cap", c_f64),
        ("window_min", c_i32), ("window_max", c_i32), ("current_step", c_i32),
        ("mode", c_i32), ("threads", c_i32),
        ("total_tokens", c_vp), ("blocks", c_vp), ("live_balance", c_vp),
        ("parked_balance", c_vp), ("forecast_live", c_vp), ("forecast_parked", c_vp),
        ("strides_out", c_vp), ("device_enumerate", c_i32),
    ]


class PlanResult(ctypes.Structure):
    """Mirror of ``ofb_plan_result``."""

    _fields_ = [("status", c_i32), ("decode_window", c_i32), ("expiry_step", c_i32),
                ("candidates_feasible", c_i64), ("candidates_priced", c_i64),
                ("candidates_ranked", c_i64), ("enumeration_windows", c_i32)]


class OprojDesc(ctypes.Structure):
    """Mirror of ``ofb_oproj_desc``."""

    _fields_ = [
        ("x", c_vp), ("w", c_vp), ("out", c_vp),
        ("layers", c_i32), ("layer", c_i32), ("batch", c_i32), ("k", c_i32), ("hidden", c_i32),
        ("workspace", c_vp), ("workspace_bytes", c_i64),
        ("world", c_i32), ("rank", c_i32), ("max_batch", c_i32),
        ("symm", c_vp * 8), ("epoch", ctypes.c_uint32), ("status", c_vp), ("timeout_ns", c_i64),
        ("w_layout", c_i32), ("residual", c_vp),
        ("out_parts", c_i32), ("part_cols", c_i32 * 4), ("part_out", c_vp * 4),
        ("ss_out", c_vp), ("ss_in", c_vp), ("ss_tiles", c_i32), ("eps", ctypes.c_float),
        ("swiglu", c_i32), ("x_layers", c_i32),
        ("kv_pool", c_vp), ("kv_tables", c_vp), ("kv_positions", c_vp), ("kv_host_slabs", c_vp),
        ("kv_max_blocks", c_i32), ("kv_part", c_i32), ("kv_block_bytes", c_i64),
    ]


# name -> (restype, argtypes); exactly the symbols include/orbitflow_b200.h declares
SIGNATURES = {
    "ofb_version": (ctypes.c_char_p, []),
    "ofb_last_error": (ctypes.c_char_p, []),
    "ofb_set_attention_kernel": (ctypes.c_int, [c_i32]),
    "ofb_k1_trace": (ctypes.c_int, [c_vp]),
    "ofb_k1_trace_sized": (ctypes.c_int, [c_vp, c_i32]),
    "ofb_attention_variant_for": (ctypes.c_int, [c_i32, c_i32, c_i32]),
    "ofb_attention_cluster_plan": (ctypes.c_int, [c_i32, c_i32, c_i32, ctypes.c_void_p, ctypes.c_void_p,
                                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ofb_attention_cluster_slots": (ctypes.c_int, [ctypes.c_void_p]),
    "ofb_attention_split_plan": (ctypes.c_int, [c_i32, c_i32, c_i32, c_i32, c_i32, c_i32,
                                                ctypes.POINTER(c_i32), ctypes.POINTER(c_i32)]),
    "ofb_attention_instep_plan": (ctypes.c_int, [c_i32, c_i32, c_i32, c_i32, c_i32, c_i32,
                                                 ctypes.POINTER(c_i32), ctypes.POINTER(c_i32),
                                                 ctypes.POINTER(c_i32)]),
    "ofb_device_info": (ctypes.c_int, [c_i32p, c_i32p]),
    "ofb_host_alloc": (c_vp, [c_i64]),
    "ofb_host_free": (ctypes.c_int, [c_vp]),
    "ofb_attention_workspace_bytes": (c_i64, [c_i32, c_i32, c_i32, c_i32]),
    "ofb_decode_attention": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_i32, c_vp, c_vp, c_i64,
                                            c_i32, c_i32, c_i32, c_i32, c_i32, c_f32, c_vp]),
    "ofb_kv_append": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_i32, c_i32, c_i32,
                                     c_i32, c_vp]),
    "ofb_kv_prefill": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_vp]),
    "ofb_runtime_create": (c_vp, [c_i32]),
    "ofb_runtime_destroy": (ctypes.c_int, [c_vp]),
    "ofb_runtime_decode_step": (ctypes.c_int, [c_vp, ctypes.POINTER(StepDesc), c_vp]),
    "ofb_runtime_step_begin": (ctypes.c_int, [c_vp, ctypes.POINTER(StepDesc), c_vp]),
    "ofb_runtime_step_layers": (ctypes.c_int, [c_vp, c_i32]),
    "ofb_runtime_step_end": (ctypes.c_int, [c_vp]),
    "ofb_runtime_step_abort": (ctypes.c_int, [c_vp]),
    "ofb_runtime_prefetch_fence": (ctypes.c_int, [c_vp, c_vp]),
    "ofb_runtime_prefetch_stats": (ctypes.c_int, [c_vp, c_i64p, c_i64p]),
    "ofb_runtime_migrate": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp]),
    "ofb_runtime_timing": (ctypes.c_int, [c_vp, ctypes.POINTER(StepTiming)]),
    "ofb_runtime_migration_pending": (ctypes.c_int, [c_vp, c_i32]),
    "ofb_runtime_timing_reset": (ctypes.c_int, [c_vp]),
    "ofb_runtime_stream_stats": (ctypes.c_int, [c_vp, c_i32, ctypes.POINTER(c_f64),
                                                ctypes.POINTER(c_f64), c_i32p]),
    "ofb_symm_alloc": (ctypes.c_int, [c_i64, ctypes.POINTER(c_vp)]),
    "ofb_symm_free": (ctypes.c_int, [c_vp]),
    "ofb_ipc_get_handle": (ctypes.c_int, [c_vp, c_vp]),
    "ofb_ipc_open_handle": (ctypes.c_int, [c_vp, ctypes.POINTER(c_vp)]),
    "ofb_ipc_close_handle": (ctypes.c_int, [c_vp]),
    "ofb_oproj_symm_bytes": (c_i64, [c_i32, c_i32, c_i32]),
    "ofb_oproj_workspace_bytes": (c_i64, [c_i32, c_i32, c_i32]),
    "ofb_oproj_allreduce": (ctypes.c_int, [ctypes.POINTER(OprojDesc), c_vp]),
    "ofb_k6_trace": (ctypes.c_int, [c_vp]),
    "ofb_rmsnorm": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_i32, ctypes.c_float, c_vp]),
    "ofb_silu_mul": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_vp]),
    "ofb_row_sumsq": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_i32, c_vp]),
    "ofb_plan_solve": (ctypes.c_int, [ctypes.POINTER(PlanProblem), ctypes.POINTER(PlanResult)]),
    "ofb_plan_last_error": (ctypes.c_char_p, []),
    "ofb_link_probe": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i32, ctypes.POINTER(c_f64),
                                      ctypes.POINTER(c_f64)]),
}


class NativeError(RuntimeError):
    """A call into the sm_100a library failed (CUDA error or bad argument)."""


def lib_path() -> Path:
    env = os.environ.get("OFB_LIB")
    if env:
        return Path(env)
    return Path(__file__).resolve().parent / "_lib" / "liborbitflow_b200.so"


def load(build_if_missing: bool = True):
    """Load (building first if needed) the library; raises if unavailable."""
    global _LIB
    with _LOCK:
        if _LIB is not None:
            return _LIB
        path = lib_path()
        if not path.exists() and build_if_missing:
            from . import build as _build

            _build.build()
        if not path.exists():
            raise NativeError(f"sm_100a library not found at {path}; run __graft_entry__.build()")
        # make sure torch's CUDA runtime is the one resolved first
        try:
            import torch  # noqa: F401
        except Exception:  # pragma: no cover - torch is always present here
            pass
        lib = ctypes.CDLL(str(path), mode=ctypes.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
        return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = _LIB.ofb_last_error().decode() if _LIB is not None else ""
        raise NativeError(f"{what} failed (rc={rc}): {msg}")
