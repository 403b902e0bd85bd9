"""Generate tests/golden/vllm_attention.npz on a GPU box: vLLM PagedAttention v2
(the kernel family the paper ran) on seeded paged KV
(tests/kvgen.make_case), so the CPU suite can pin the attention oracle against
it without a GPU (tests/test_oracle.py).

    python tests/golden/make_vllm_attention_golden.py     # needs CUDA + vllm._C
"""
import sys
from pathlib import Path

import numpy as np
import torch

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from kvgen import bf16_bits, make_case  # noqa: E402

CASES = [  # (seq_lens, hq, hkv, seed)
    ([700, 33, 1, 255], 8, 2, 101),        # toy heads, ragged, partial blocks
    ([1000, 17], 32, 8, 102),              # Llama-3.1-8B heads (group 4)
    ([513, 64], 64, 8, 103),               # Llama-3.1-70B heads (group 8)
    ([900], 8, 1, 104),                    # 70B TP8 shard (1 KV head, group 8)
    ([300, 129], 16, 1, 105),              # group 16 (max)
]


def main():
    from vllm import _custom_ops as ops

    dev = torch.device("cuda:0")
    out = {}
    for i, (lens, hq, hkv, seed) in enumerate(CASES):
        case = make_case(lens, hq, hkv, seed=seed)
        pool = case["pool"].to(dev)
        nblk = pool.shape[0]
        key_cache = pool[:, :, 0].reshape(nblk, hkv, 16, 16, 8).permute(0, 1, 3, 2, 4).contiguous()
        value_cache = pool[:, :, 1].permute(0, 1, 3, 2).contiguous()
        q = case["q"].to(dev)
        o = torch.empty_like(q)
        max_len = max(lens)
        nparts = (max_len + 511) // 512
        exp_sums = torch.empty((len(lens), hq, nparts), dtype=torch.float32, device=dev)
        max_logits = torch.empty_like(exp_sums)
        tmp = torch.empty((len(lens), hq, nparts, 128), dtype=q.dtype, device=dev)
        one = torch.ones((), dtype=torch.float32, device=dev)
        ops.paged_attention_v2(o, exp_sums, max_logits, tmp, q, key_cache, value_cache, hkv,
                               case["scale"], torch.from_numpy(case["block_tables"]).to(dev),
                               torch.from_numpy(case["seq_lens"]).to(dev), 16, max_len, None,
                               "auto", one, one)
        torch.cuda.synchronize()
        out[f"case{i}_out"] = bf16_bits(o.cpu())
        out[f"case{i}_meta"] = np.array([hq, hkv, seed] + list(lens), dtype=np.int64)
    np.savez_compressed(HERE / "vllm_attention.npz", **out)
    print("wrote", HERE / "vllm_attention.npz", sorted(out))


if __name__ == "__main__":
    main()
