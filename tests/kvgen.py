"""Seeded synthetic paged-KV inputs shared by the parity tests.

Values are N(0,1) bf16 drawn from a CPU ``torch.Generator`` so the oracle and
the GPU see identical bits.  Block tables are a random
permutation of pool blocks, i.e. genuinely paged (non-contiguous) slabs.
"""

from __future__ import annotations

import math

import numpy as np
import torch

BLOCK = 16
D = 128


def bf16_bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).numpy().view(np.uint16)


def make_case(seq_lens, hq, hkv, seed=0, spare_blocks=3, max_blocks=None):
    g = torch.Generator().manual_seed(seed)
    b = len(seq_lens)
    nblk = [(s + BLOCK - 1) // BLOCK for s in seq_lens]
    total = sum(nblk) + spare_blocks
    width = max_blocks or max(1, max(nblk))
    pool = torch.randn((max(total, 1), hkv, 2, BLOCK, D), generator=g).to(torch.bfloat16)
    q = torch.randn((b, hq, D), generator=g).to(torch.bfloat16)
    perm = torch.randperm(max(total, 1), generator=g).numpy().astype(np.int32)
    bt = np.full((b, width), -1, dtype=np.int32)
    cur = 0
    for i, n in enumerate(nblk):
        bt[i, :n] = perm[cur:cur + n]
        cur += n
    return {
        "q": q, "pool": pool, "block_tables": bt,
        "seq_lens": np.asarray(seq_lens, dtype=np.int32),
        "scale": 1.0 / math.sqrt(D), "hq": hq, "hkv": hkv,
    }
