"""B200 calibration of the reference cost model (``SystemProfile``).

The reference's profile is a desk calibration (``defaults.py``):
per-layer compute linear in batch tokens and one bandwidth in blocks/ms.  On
B200 both terms come from measurements of this repo's kernels:

* ``compute_per_token_ms`` = KV bytes per token per layer / achieved K1 HBM
  bandwidth (K1 streams every cached token once);
* ``compute_base_ms``      = per-layer fixed cost (launch + pipeline fill of K1,
  K3 and the per-layer waits), measured on short contexts;
* ``bandwidth_blocks_per_ms`` = measured pinned H2D GB/s / block bytes.

Block bytes follow the served shape: 16 tokens x Hkv x 2 x 128 x 2 B
(64 KiB for Llama-3.1-8B, 64/TP KiB per GPU for the 70B shape).
"""

from __future__ import annotations

from .core import SystemProfile

# Round-1 B200 measurements (profiles/r01_summary.md): K1 at 6.40 TB/s on
# 32K-token contexts; host link 55.6 GB/s H2D; ~12 us fixed per layer.
B200_K1_GBS = 6400.0
B200_H2D_GBS = 55.6
B200_LAYER_FIXED_MS = 0.012


def b200_profile(num_layers: int, num_kv_heads: int, gpu_block_budget: int, *,
                 k1_gbs: float = B200_K1_GBS, h2d_gbs: float = B200_H2D_GBS,
                 layer_fixed_ms: float = B200_LAYER_FIXED_MS, head_dim: int = 128,
                 block_size: int = 16, prefill_per_token_ms: float = 0.0002) -> SystemProfile:
    kv_bytes_per_token = num_kv_heads * 2 * head_dim * 2
    block_bytes = kv_bytes_per_token * block_size
    return SystemProfile(
        num_layers=num_layers,
        compute_base_ms=layer_fixed_ms,
        compute_per_token_ms=kv_bytes_per_token / (k1_gbs * 1e6),
        bandwidth_blocks_per_ms=h2d_gbs * 1e6 / block_bytes,
        gpu_block_budget=gpu_block_budget,
        block_size=block_size,
        prefill_per_token_ms=prefill_per_token_ms,
    )


def measure_b200_profile(num_layers: int, num_q_heads: int, num_kv_heads: int,
                         gpu_block_budget: int, *, batch: int = 16,
                         contexts: tuple[int, int] = (2048, 16384), iters: int = 10,
                         device=None) -> tuple[SystemProfile, dict]:
    """Calibrate the cost model on this GPU instead of using the round-1 constants
    (SURVEY.md H4): time K1 (CUDA events, back-to-back launches) on synthetic paged
    KV at two context lengths - slope -> ``compute_per_token_ms``, intercept ->
    ``compute_base_ms`` - and probe the pinned host link (best-of-10 1 GiB H2D) for
    ``bandwidth_blocks_per_ms``.  Returns the profile and the raw measurements."""
    import statistics

    import torch

    from . import _native, ops
    from .runtime import link_probe

    dev = torch.device(device if device is not None else "cuda")
    times = {}
    for ctx in contexts:
        nblk = (ctx + 15) // 16
        pools = [torch.empty((batch * nblk, num_kv_heads, 2, 16, 128), dtype=torch.bfloat16,
                             device=dev).normal_() for _ in range(2)]
        bt = torch.arange(batch * nblk, dtype=torch.int32, device=dev).reshape(batch, nblk)
        lens = torch.full((batch,), ctx, dtype=torch.int32, device=dev)
        q = torch.randn((batch, num_q_heads, 128), device=dev).to(torch.bfloat16)
        out = torch.empty_like(q)
        ws = ops.workspace(batch, num_q_heads, num_kv_heads, ctx, dev)
        for p in pools:
            ops.decode_attention(q, p, bt, lens, out=out, max_seq_len=ctx, ws=ws)
        torch.cuda.synchronize()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(iters + 1)]
        evs[0].record()
        for i in range(iters):
            ops.decode_attention(q, pools[i % 2], bt, lens, out=out, max_seq_len=ctx, ws=ws)
            evs[i + 1].record()
        torch.cuda.synchronize()
        times[ctx] = statistics.median(evs[i].elapsed_time(evs[i + 1]) for i in range(iters))
        del pools
    (c0, t0), (c1, t1) = sorted(times.items())
    per_token = (t1 - t0) / ((c1 - c0) * batch)          # ms per cached token per layer
    base = max(t0 - per_token * c0 * batch, 0.0)
    lib = _native.load()
    nbytes = 1 << 30
    host = lib.ofb_host_alloc(nbytes)
    if not host:
        raise RuntimeError("pinned probe buffer allocation failed")
    try:
        d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        h2d, d2h = link_probe(host, d.data_ptr(), nbytes, 10)
    finally:
        lib.ofb_host_free(host)
    kv_bytes_per_token = num_kv_heads * 2 * 128 * 2
    k1_gbs = kv_bytes_per_token / (per_token * 1e6)
    prof = b200_profile(num_layers, num_kv_heads, gpu_block_budget, k1_gbs=k1_gbs, h2d_gbs=h2d,
                        layer_fixed_ms=base)
    return prof, {"k1_ms": times, "k1_gbs_slope": k1_gbs, "layer_fixed_ms": base,
                  "h2d_gbs": h2d, "d2h_gbs": d2h}
