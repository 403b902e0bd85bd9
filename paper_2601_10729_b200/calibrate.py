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
