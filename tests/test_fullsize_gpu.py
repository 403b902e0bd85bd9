"""Parity at BASELINE.json's full sizes (SURVEY.md 8(d) cfg2 / cfg4 shapes).

The full-size KV (2 GiB per 8B layer, 1 GiB per 70B TP8 shard layer) is
generated on the GPU; the CPU oracle checks sampled requests exactly as
loaded back from HBM, and size-independent properties cover the rest:

* V linearity: doubling every V row (exact in bf16) doubles the output
  bit for bit - every op on the V path (HMMA accumulate, split combine,
  normalisation, bf16 rounding) commutes with a power-of-two scale;
* placement independence: moving every block to another pool address (the
  table follows) gives a bit-identical output - the work decomposition
  depends only on logical (request, head, block) order, never on where a
  block lives (the executor relies on this when it restores a slab to a new
  extent);
* the full cfg2 step (B=16, 32K context, 8B heads, stride-2 plan) moves
  exactly ``blocks_to_fetch`` blocks and every output matches the oracle.

Tolerance (north_star): 2e-2 relative / 1e-2 absolute, bf16 vs the oracle.
"""

import math

import numpy as np
import pytest
import torch

import oracle
from kvgen import BLOCK, D, bf16_bits

pytestmark = pytest.mark.gpu

RTOL, ATOL = 2e-2, 1e-2
SCALE = 1.0 / math.sqrt(D)


@pytest.fixture(params=["stream", "split"])
def k1_variant(request):
    from paper_2601_10729_b200 import ops

    prev = ops.set_attention_kernel(request.param)
    yield request.param
    ops.set_attention_kernel(prev)


def _device_case(batch, tokens, hq, hkv, seed):
    """Full-size paged case generated on cuda:0; slabs scattered over the pool."""
    dev = torch.device("cuda:0")
    nblk = (tokens + BLOCK - 1) // BLOCK
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    pool = torch.randn((batch * nblk + 7, hkv, 2, BLOCK, D), generator=g, device=dev,
                       dtype=torch.float32).to(torch.bfloat16)
    q = torch.randn((batch, hq, D), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    perm = torch.randperm(pool.shape[0], generator=g, device=dev)[: batch * nblk]
    tables = perm.view(batch, nblk).to(torch.int32).contiguous()
    lens = torch.full((batch,), tokens, dtype=torch.int32, device=dev)
    return pool, q, tables, lens


def _attend(pool, q, tables, lens, max_len):
    from paper_2601_10729_b200 import ops

    out = ops.decode_attention(q, pool, tables, lens, max_seq_len=max_len, scale=SCALE)
    torch.cuda.synchronize()
    return out


def _oracle_rows(pool, q, tables, lens, rows):
    """Oracle output for sampled requests, from the bits actually in HBM."""
    want = {}
    for r in rows:
        n = (int(lens[r]) + BLOCK - 1) // BLOCK
        sub = pool[tables[r, :n].long()].cpu()
        bt = np.arange(n, dtype=np.int32)[None, :]
        want[r] = oracle.decode_attention(bf16_bits(q[r:r + 1].cpu()), bf16_bits(sub), bt,
                                          np.array([int(lens[r])], dtype=np.int32), SCALE)[0]
    return want


@pytest.mark.parametrize("name,batch,tokens,hq,hkv", [
    ("cfg2 8B layer", 16, 32761, 32, 8),
    ("cfg4 70B TP8 shard", 32, 65529, 8, 1),
    ("cfg4 70B TP4 shard", 32, 65529, 16, 2),
])
def test_full_size_layer_sampled_and_properties(k1_variant, name, batch, tokens, hq, hkv):
    pool, q, tables, lens = _device_case(batch, tokens, hq, hkv, seed=batch + hq)
    out = _attend(pool, q, tables, lens, tokens)
    assert torch.isfinite(out.float()).all(), name
    rows = [0, batch // 2 + 1, batch - 1]
    want = _oracle_rows(pool, q, tables, lens, rows)
    got = out.float().cpu().numpy()
    for r in rows:
        np.testing.assert_allclose(got[r], want[r], rtol=RTOL, atol=ATOL, err_msg=f"{name} request {r}")

    # V linearity, bit for bit
    pool2 = pool.clone()
    pool2[:, :, 1] *= 2
    out2 = _attend(pool2, q, tables, lens, tokens)
    assert torch.equal(out2, out * 2), f"{name}: out(2V) != 2 out(V)"
    del pool2

    # placement independence: every block moved, table follows, output identical
    dev = pool.device
    g = torch.Generator(device=dev)
    g.manual_seed(11)
    move = torch.randperm(pool.shape[0], generator=g, device=dev)
    pool3 = torch.empty_like(pool)
    pool3[move] = pool
    tables3 = move[tables.long()].to(torch.int32)
    out3 = _attend(pool3, q, tables3, lens, tokens)
    assert torch.equal(out3, out), f"{name}: output depends on block addresses"


def test_full_size_cfg2_step_fetch_volume_and_outputs():
    """The cfg2 step at full B and context (4 of the 32 layers, same stride-2
    plan): fetched bytes == blocks_to_fetch x block bytes, every (layer,
    request) output vs the oracle, and the offloaded layers' host slabs hold
    the appended token (K3 writes it through the mapped host slot)."""
    from paper_2601_10729_b200.core import PlacementMatrix, RequestState
    from paper_2601_10729_b200.executor import B200Executor, ModelShape
    from paper_2601_10729_b200.latency import blocks_to_fetch

    shape = ModelShape(4, 32, 8)
    B, prompt = 16, 32760
    batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=prompt, target_output_tokens=8)
             for i in range(B)]
    placement = PlacementMatrix.from_strides(range(B), shape.num_layers, [2] * B)
    assert all(row == (1, 0, 1, 0) for row in placement.rows)
    cap = -(-(prompt + 8 + 1) // BLOCK)
    ex = B200Executor(shape, device_blocks=B * 2 * cap + B * 2 * cap + 16, host_blocks=B * 2 * cap + 16,
                      staging_slots=2, record_timing=True, seed=5)
    try:
        ex.install(batch, placement)
        for _step in range(2):
            ex.decode_step(batch, placement)
            t = ex.last_timing
            assert t["copy_bytes"] == blocks_to_fetch(placement, batch) * shape.block_bytes
            assert t["copies"] == B * 2 and t["layers"] == 4
            pos = ex.last_positions
            out = ex.last_output.float().cpu().numpy()
            k_new = ex.last_inputs["k_new"]
            v_new = ex.last_inputs["v_new"]
            for layer in range(4):
                for b, r in enumerate(batch):
                    n = int(pos[b]) // BLOCK + 1
                    slab = ex.slab_bits(r.id, layer, n)
                    qb = bf16_bits(ex.last_inputs["q"][layer, b:b + 1].cpu())
                    want = oracle.decode_attention(qb, slab, np.arange(n, dtype=np.int32)[None, :],
                                                   np.array([pos[b] + 1], dtype=np.int32), SCALE)[0]
                    np.testing.assert_allclose(out[layer, b], want, rtol=RTOL, atol=ATOL,
                                               err_msg=f"layer {layer} request {r.id}")
                    # the new token landed at slot pos of the slab (host or HBM)
                    blk, slot = divmod(int(pos[b]), BLOCK)
                    np.testing.assert_array_equal(slab[blk, :, 0, slot], bf16_bits(k_new[layer, b].cpu()))
                    np.testing.assert_array_equal(slab[blk, :, 1, slot], bf16_bits(v_new[layer, b].cpu()))
            for r in batch:
                r.record_generated_token()
    finally:
        ex.close()
