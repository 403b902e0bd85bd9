"""K1 (paged GQA decode attention) and K3 (append) on the GPU vs the CPU oracle.

Tolerance (BASELINE.json north_star): bf16 GPU output vs the fp32/f64 CPU
oracle within 2e-2 relative / 1e-2 absolute.  The append is byte work and is
checked bit-exactly.
"""

import numpy as np
import pytest
import torch

import oracle
from kvgen import BLOCK, D, bf16_bits, make_case

pytestmark = pytest.mark.gpu

RTOL, ATOL = 2e-2, 1e-2


@pytest.fixture(params=["stream", "split", "split2", "cluster", "auto"], autouse=True)
def k1_variant(request):
    """Every K1 parity test runs under every work decomposition (stream-K, split
    with the in-kernel combine, split with the separate combine kernel, cluster)
    and under the auto policy."""
    from paper_2601_10729_b200 import ops

    prev = ops.set_attention_kernel(request.param)
    yield request.param
    ops.set_attention_kernel(prev)


_BINDING = ["ctypes"]


@pytest.fixture(params=["ctypes", "torch"], autouse=True)
def binding(request):
    """...and through both bindings: the ctypes C ABI and torch.ops.orbit."""
    _BINDING[0] = request.param
    yield request.param
    _BINDING[0] = "ctypes"


def _run_gpu(case, max_seq_len=None):
    from paper_2601_10729_b200 import ops, torch_ops

    dev = torch.device("cuda:0")
    args = (case["q"].to(dev), case["pool"].to(dev),
            torch.from_numpy(case["block_tables"]).to(dev),
            torch.from_numpy(case["seq_lens"]).to(dev))
    if _BINDING[0] == "torch":
        msl = max_seq_len if max_seq_len is not None else int(case["seq_lens"].max(initial=0))
        out = torch_ops.decode_attention(*args, msl, scale=case["scale"])
    else:
        out = ops.decode_attention(*args, max_seq_len=max_seq_len, scale=case["scale"])
    torch.cuda.synchronize()
    return out.float().cpu().numpy()


def _run_oracle(case):
    return oracle.decode_attention(bf16_bits(case["q"]), bf16_bits(case["pool"]),
                                   case["block_tables"], case["seq_lens"], case["scale"])


@pytest.mark.parametrize("seq_lens,hq,hkv", [
    ([4088, 4088, 4088, 4088], 8, 2),          # cfg1 toy shape (group 4)
    ([4089, 17, 1, 300], 8, 2),                  # ragged, partial last blocks
    ([1000, 2048], 32, 8),                       # Llama-3.1-8B heads (group 4)
    ([3000, 5], 64, 8),                          # Llama-3.1-70B heads (group 8)
    ([777], 16, 1),                              # group 16 (max)
    ([513, 64], 4, 4),                           # MHA (group 1)
    # long single requests: many splits, so the combine runs with 5 / 2 / 1
    # thread groups dealing the splits (groups 1 / 2 / 16)
    ([20000, 3], 2, 2),
    ([24001], 4, 2),
    ([30000, 700], 16, 1),
])
def test_attention_matches_oracle(seq_lens, hq, hkv):
    case = make_case(seq_lens, hq, hkv, seed=sum(seq_lens) + hq)
    got = _run_gpu(case)
    want = _run_oracle(case)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


def test_long_context_many_splits_and_rearm():
    # 40K tokens on one (request, head): dozens of splits, last-CTA combine;
    # a second launch checks that the split counters re-armed themselves.
    case = make_case([40000, 31], 4, 1, seed=7)
    first = _run_gpu(case)
    second = _run_gpu(case)
    want = _run_oracle(case)
    np.testing.assert_allclose(first, want, rtol=RTOL, atol=ATOL)
    np.testing.assert_array_equal(first, second)


def test_empty_request_gives_zeros():
    case = make_case([0, 100], 8, 2, seed=3)
    got = _run_gpu(case, max_seq_len=100)
    assert np.all(got[0] == 0.0)
    np.testing.assert_allclose(got[1], _run_oracle(case)[1], rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("positions", [[4088, 17, 0, 300], [15, 16, 31, 47]])
def test_append_bit_exact(positions):
    from paper_2601_10729_b200 import ops, torch_ops

    hkv, b = 2, len(positions)
    case = make_case([p + 1 for p in positions], 8, hkv, seed=5)
    g = torch.Generator().manual_seed(99)
    k_new = torch.randn((b, hkv, D), generator=g).to(torch.bfloat16)
    v_new = torch.randn((b, hkv, D), generator=g).to(torch.bfloat16)
    pos = np.asarray(positions, dtype=np.int32)

    want = bf16_bits(case["pool"]).copy()
    oracle.kv_append(bf16_bits(k_new), bf16_bits(v_new), want, case["block_tables"], pos)

    dev = torch.device("cuda:0")
    pool = case["pool"].to(dev)
    append = torch_ops.kv_append if _BINDING[0] == "torch" else ops.kv_append
    append(k_new.to(dev), v_new.to(dev), pool, torch.from_numpy(case["block_tables"]).to(dev),
           torch.from_numpy(pos).to(dev))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(bf16_bits(pool.cpu()), want)


def test_append_then_attend_sees_new_token():
    from paper_2601_10729_b200 import ops

    case = make_case([4096, 34], 8, 2, seed=21)
    g = torch.Generator().manual_seed(5)
    k_new = torch.randn((2, 2, D), generator=g).to(torch.bfloat16)
    v_new = torch.randn((2, 2, D), generator=g).to(torch.bfloat16)
    pos = np.asarray([4095, 33], dtype=np.int32)  # slot 15 of block 255; slot 1 of block 2
    dev = torch.device("cuda:0")
    pool = case["pool"].to(dev)
    bt = torch.from_numpy(case["block_tables"]).to(dev)
    ops.kv_append(k_new.to(dev), v_new.to(dev), pool, bt, torch.from_numpy(pos).to(dev))
    lens = torch.from_numpy(pos + 1).to(dev)
    got = ops.decode_attention(case["q"].to(dev), pool, bt, lens, scale=case["scale"])
    torch.cuda.synchronize()
    host_pool = bf16_bits(case["pool"]).copy()
    oracle.kv_append(bf16_bits(k_new), bf16_bits(v_new), host_pool, case["block_tables"], pos)
    want = oracle.decode_attention(bf16_bits(case["q"]), host_pool, case["block_tables"], pos + 1,
                                   case["scale"])
    np.testing.assert_allclose(got.float().cpu().numpy(), want, rtol=RTOL, atol=ATOL)


def test_garbage_past_sequence_end_is_ignored():
    # NaN bit patterns in the unused slots of the last block must not leak
    # into the output (P is 0 there, but 0 * NaN = NaN in a P.V tile).
    case = make_case([33, 16 * 5 + 1, 7], 8, 2, seed=9)
    pool = case["pool"].clone()
    bits = pool.view(torch.int16)
    for b, seq in enumerate(case["seq_lens"]):
        blk = case["block_tables"][b][(seq - 1) // 16]
        bits[blk, :, :, (seq % 16 or 16):, :] = 0x7FC0          # bf16 quiet NaN
    case["pool"] = pool
    got = _run_gpu(case)
    assert not np.isnan(got).any()
    np.testing.assert_allclose(got, _run_oracle(case), rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("seed", [0, 1])
def test_ragged_batch_with_empty_and_tiny_requests(seed):
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, 3000, size=37)
    lens[[3, 11, 20]] = 0
    lens[[5, 6]] = 1
    lens[7] = 16
    lens[8] = 17
    case = make_case(lens.tolist(), 8, 2, seed=seed)
    got = _run_gpu(case, max_seq_len=int(lens.max()))
    want = _run_oracle(case)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


def test_one_pair_spans_every_cta():
    case = make_case([100_000], 4, 1, seed=4)     # 6250 tiles over the whole grid
    np.testing.assert_allclose(_run_gpu(case), _run_oracle(case), rtol=RTOL, atol=ATOL)


def test_max_seq_len_overestimate_and_tiny_work():
    case = make_case([5, 3], 8, 2, seed=6, max_blocks=4096)   # W = 2 tiles, grid sized for 64K
    got = _run_gpu(case, max_seq_len=65536)
    np.testing.assert_allclose(got, _run_oracle(case), rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("tokens", [1, 16, 37, 300])
def test_prefill_writes_paged_layout_to_device_and_host(tokens):
    """K5 scatters token-major prompt K/V into the paged block layout, to an HBM
    extent and to a mapped pinned host slab alike (bit-exact)."""
    from paper_2601_10729_b200 import ops
    from paper_2601_10729_b200.kvpool import HostArena

    L, hkv = 3, 2
    nblk = (tokens + 15) // 16
    g = torch.Generator().manual_seed(tokens)
    k = torch.randn((L, tokens, hkv, D), generator=g).to(torch.bfloat16)
    v = torch.randn((L, tokens, hkv, D), generator=g).to(torch.bfloat16)
    dev = torch.device("cuda:0")
    pool = torch.zeros((2 * nblk, hkv, 2, 16, D), dtype=torch.bfloat16, device=dev)
    block_bytes = hkv * 8192
    arena = HostArena(nblk, block_bytes)
    try:
        dsts = [pool.data_ptr(), pool.data_ptr() + nblk * block_bytes, arena.base]
        ops.kv_prefill(k.to(dev), v.to(dev), torch.tensor(dsts, dtype=torch.int64).to(dev))
        torch.cuda.synchronize()
        slabs = [bf16_bits(pool[:nblk].cpu()), bf16_bits(pool[nblk:].cpu()),
                 arena.view_u16(0, nblk).reshape(nblk, hkv, 2, 16, D).copy()]
        for l in range(L):
            for t in range(tokens):
                for h in range(hkv):
                    np.testing.assert_array_equal(slabs[l][t // 16, h, 0, t % 16], bf16_bits(k[l, t, h]))
                    np.testing.assert_array_equal(slabs[l][t // 16, h, 1, t % 16], bf16_bits(v[l, t, h]))
    finally:
        arena.close()
