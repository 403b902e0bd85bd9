"""Attention parity anchored on vLLM's PagedAttention kernel.

The paper's attention is vLLM v0.6.6 PagedAttention (PAPER.md:202, :367,
:750); kvsim itself has no attention.  The image ships vLLM
0.22, whose ``paged_attention_v1`` / ``_v2`` are the same PagedAttention
kernels (16-token blocks, GQA through num_kv_heads).  This test runs them on
the same seeded paged KV as the CPU oracle and K1: oracle vs vLLM pins the
oracle's semantics to the implementation the paper ran; K1 vs vLLM checks the
product against it directly.  vLLM is only the checker here (test code).

Tolerance: 2e-2 relative / 1e-2 absolute (bf16 outputs, BASELINE north_star).
"""

import numpy as np
import pytest
import torch

import oracle
from kvgen import bf16_bits, make_case

pytestmark = pytest.mark.gpu

RTOL, ATOL = 2e-2, 1e-2


def _vllm_ops():
    try:
        from vllm import _custom_ops as ops

        if not hasattr(torch.ops, "_C") or not hasattr(torch.ops._C, "paged_attention_v1"):
            pytest.skip("vllm._C (PagedAttention kernels) not loadable on this box")
        return ops
    except Exception as exc:  # pragma: no cover - depends on the image
        pytest.skip(f"vllm not importable: {exc!r}")


def _vllm_layout(pool: torch.Tensor):
    """[blocks, Hkv, 2, 16, 128] -> vLLM key_cache [blocks, Hkv, 128/8, 16, 8] and
    value_cache [blocks, Hkv, 128, 16] (bf16: x = 16 bytes / 2)."""
    nblk, hkv = pool.shape[0], pool.shape[1]
    k = pool[:, :, 0]
    v = pool[:, :, 1]
    key_cache = k.reshape(nblk, hkv, 16, 16, 8).permute(0, 1, 3, 2, 4).contiguous()
    value_cache = v.permute(0, 1, 3, 2).contiguous()
    return key_cache, value_cache


@pytest.mark.parametrize("version", ["v1", "v2"])
@pytest.mark.parametrize("seq_lens,hq,hkv", [
    ([4088, 4088, 4088, 4088], 8, 2),     # cfg1 toy shape
    ([4089, 17, 1, 300], 8, 2),             # ragged, partial last blocks
    ([1000, 2048], 32, 8),                  # Llama-3.1-8B heads
    ([3000, 5], 64, 8),                     # Llama-3.1-70B heads
    ([9000], 8, 1),                         # 70B TP8 shard (one KV head, group 8)
])
def test_oracle_and_k1_agree_with_vllm_paged_attention(version, seq_lens, hq, hkv):
    ops = _vllm_ops()
    from paper_2601_10729_b200 import ops as ofb

    dev = torch.device("cuda:0")
    case = make_case(seq_lens, hq, hkv, seed=sum(seq_lens) + hq + 1)
    q = case["q"].to(dev)
    pool = case["pool"].to(dev)
    bt = torch.from_numpy(case["block_tables"]).to(dev)
    lens = torch.from_numpy(case["seq_lens"]).to(dev)
    max_len = int(max(seq_lens))
    key_cache, value_cache = _vllm_layout(pool)
    out = torch.empty_like(q)
    one = torch.ones((), dtype=torch.float32, device=dev)
    if version == "v1":
        ops.paged_attention_v1(out, q, key_cache, value_cache, hkv, case["scale"], bt, lens, 16,
                               max_len, None, "auto", one, one)
    else:
        part = 512
        nparts = (max_len + part - 1) // part
        exp_sums = torch.empty((len(seq_lens), hq, nparts), dtype=torch.float32, device=dev)
        max_logits = torch.empty_like(exp_sums)
        tmp = torch.empty((len(seq_lens), hq, nparts, 128), dtype=q.dtype, device=dev)
        ops.paged_attention_v2(out, exp_sums, max_logits, tmp, q, key_cache, value_cache, hkv,
                               case["scale"], bt, lens, 16, max_len, None, "auto", one, one)
    ours = ofb.decode_attention(q, pool, bt, lens, max_seq_len=max_len, scale=case["scale"])
    torch.cuda.synchronize()
    vllm_out = out.float().cpu().numpy()
    want = oracle.decode_attention(bf16_bits(case["q"]), bf16_bits(case["pool"]),
                                   case["block_tables"], case["seq_lens"], case["scale"])
    np.testing.assert_allclose(want, vllm_out, rtol=RTOL, atol=ATOL, err_msg="oracle vs vLLM")
    np.testing.assert_allclose(ours.float().cpu().numpy(), vllm_out, rtol=RTOL, atol=ATOL,
                               err_msg="K1 vs vLLM")
