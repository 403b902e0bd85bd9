"""The C-ABI library builds, loads and exports exactly what include/*.h declares.

CPU-only: no compute calls (there is no GPU in the build container)."""

import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    text = (ROOT / "include" / "orbitflow_b200.h").read_text()
    return sorted(set(re.findall(r"OFB_API[^;(]*?\b(ofb_\w+)\s*\(", text, re.S)))


def test_header_declares_the_boundary():
    names = _declared()
    for want in ("ofb_decode_attention", "ofb_kv_append", "ofb_runtime_decode_step",
                 "ofb_runtime_migrate", "ofb_host_alloc"):
        assert want in names


def test_library_exports_every_declared_symbol():
    from paper_2601_10729_b200 import _native, build

    path = build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", str(path)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (ofb_\w+)", out))
    assert set(_declared()) <= exported
    assert set(_native.SIGNATURES) == set(_declared())


def test_library_loads_and_binds():
    from paper_2601_10729_b200 import _native

    lib = _native.load()
    assert lib.ofb_version().decode().startswith("orbitflow-b200")
    # workspace sizing is host arithmetic, safe without a GPU
    assert lib.ofb_attention_workspace_bytes(16, 32, 8, 32768) > 0


def test_sm100a_sass_present():
    from paper_2601_10729_b200 import build

    path = build.build()
    sass = subprocess.run(["cuobjdump", "-sass", str(path)], capture_output=True, text=True).stdout
    assert "UTMALDG" in sass          # TMA tile loads
    assert "HMMA" in sass             # tensor-core tiles of the GQA group
    assert "LDSM" in sass


def test_sm100a_sass_has_tcgen05_in_k6():
    """K6 issues 5th-gen tensor-core MMAs (UTCHMMA), reads the accumulator from
    TMEM (LDTM) and stages operands with 3-D / 4-D TMA."""
    from paper_2601_10729_b200 import build

    path = build.build()
    sass = subprocess.run(["cuobjdump", "-sass", str(path)], capture_output=True, text=True).stdout
    for op in ("UTCHMMA", "LDTM", "UTMALDG.3D", "UTMALDG.4D"):
        assert op in sass, op


def test_k6_host_sizing_and_argument_errors():
    """Host arithmetic and argument validation of the C1 entry points (no GPU)."""
    import ctypes

    from paper_2601_10729_b200 import _native

    lib = _native.load()
    # inbox [2][world][hidden][max_batch] bf16 (256-aligned) + flags [2][world][hidden/128] u32
    inbox = 2 * 8 * 8192 * 32 * 2
    assert lib.ofb_oproj_symm_bytes(8, 32, 8192) == (inbox + 255) // 256 * 256 + 2 * 8 * 64 * 4
    assert lib.ofb_oproj_symm_bytes(9, 32, 8192) == -1          # world > 8
    assert lib.ofb_oproj_symm_bytes(2, 0, 8192) == -1
    assert lib.ofb_oproj_workspace_bytes(32, 1024, 8192) > 0
    assert lib.ofb_oproj_workspace_bytes(32, 32, 8192) == -1      # k < 64

    def call(**kw):
        d = _native.OprojDesc()
        d.x = d.w = d.out = d.workspace = 1 << 20
        d.layers, d.layer, d.batch, d.k, d.hidden = 2, 0, 8, 128, 256
        d.workspace_bytes = 256
        d.world, d.rank, d.max_batch, d.epoch, d.w_layout = 1, 0, 8, 1, 1
        for k, v in kw.items():
            setattr(d, k, v)
        rc = lib.ofb_oproj_allreduce(ctypes.byref(d), None)
        return rc, lib.ofb_last_error().decode()

    for bad, msg in [(dict(batch=9), "max_batch"), (dict(k=96), "multiple of 64"),
                     (dict(hidden=200), "multiple of 128"), (dict(layer=2), "layer"),
                     (dict(world=2, rank=0, epoch=0), "epoch"), (dict(w_layout=3), "w_layout"),
                     (dict(world=9), "world"),
                     # decoder-layer epilogues
                     (dict(ss_in=1 << 20, ss_tiles=0), "ss_in"), (dict(ss_in=1 << 20, ss_tiles=2, eps=-1.0), "ss_in"),
                     (dict(swiglu=1, residual=1 << 20), "swiglu"),
                     (dict(out_parts=2, ss_out=1 << 20), "ss_out excludes"),
                     (dict(x_layers=2), "x_layers"),
                     (dict(kv_pool=1 << 20), "kv_pool")]:
        rc, err = call(**bad)
        assert rc == -1 and msg in err, (bad, rc, err)


def test_gate_up_interleave_round_trip():
    """The SwiGLU epilogue's weight order: rows interleaved per 64 (gate, up) and back."""
    import torch

    from paper_2601_10729_b200.collective import deinterleave_gate_up, interleave_gate_up

    w = torch.arange(2 * 2 * 192 * 3, dtype=torch.float32).reshape(2, 2 * 192, 3)
    v = interleave_gate_up(w)
    assert torch.equal(v[:, 64:128], w[:, 192:256])          # tile 0: gate 0..63 then up 0..63
    assert torch.equal(v[:, 128:192], w[:, 64:128])
    assert torch.equal(deinterleave_gate_up(v), w)


def test_runtime_calls_without_a_runtime_fail_cleanly():
    from paper_2601_10729_b200 import _native

    lib = _native.load()
    assert lib.ofb_runtime_prefetch_fence(None, None) == -1
    assert "null runtime" in lib.ofb_last_error().decode()
    assert lib.ofb_runtime_step_layers(None, 1) == -1


# (batch, hq, hkv, context) -> split length the K1 plan picks; on the B200 box
# (tools/k1_bps_sweep.py, profiles/r01_k1_bps_sweep.jsonl, 8..256 swept) each is
# within 2% of the fastest measured length for that shape
_K1_BEST_BPS = {
    (1, 8, 1, 4096): 8, (1, 8, 1, 16384): 16, (1, 8, 1, 65536): 32,
    (4, 8, 1, 4096): 8, (4, 8, 1, 16384): 32, (4, 8, 1, 65536): 64,
    (16, 8, 1, 4096): 16, (16, 8, 1, 16384): 64, (16, 8, 1, 65536): 256,
    (1, 32, 8, 4096): 16, (1, 32, 8, 16384): 32, (1, 32, 8, 65536): 128,
    (4, 32, 8, 4096): 32, (4, 32, 8, 16384): 128, (4, 32, 8, 65536): 256,
    (1, 64, 8, 4096): 16, (1, 64, 8, 16384): 32, (1, 64, 8, 65536): 128,
    (1, 16, 1, 4096): 16, (1, 16, 1, 16384): 32, (1, 16, 1, 65536): 64,
}


def _split_plan(lib, b, hq, hkv, seq, sms=148, occ=2):
    import ctypes

    bps, ns = ctypes.c_int32(), ctypes.c_int32()
    assert lib.ofb_attention_split_plan(b, hq, hkv, seq, sms, occ, ctypes.byref(bps), ctypes.byref(ns)) == 0
    return bps.value, ns.value


def test_k1_split_plan_matches_measured_best():
    """The split K1's cost model (host arithmetic, no GPU) picks, on every swept
    latency-bound shape, a split length the B200 sweep measured within 2% of the
    fastest."""
    from paper_2601_10729_b200 import _native

    lib = _native.load()
    for (b, hq, hkv, seq), best in _K1_BEST_BPS.items():
        assert _split_plan(lib, b, hq, hkv, seq)[0] == best, (b, hq, hkv, seq)


def test_k1_split_plan_invariants():
    """Every plan covers the context within the kernel's limits (<= 256 splits of
    <= 256 blocks), and a large step shape keeps the longest splits."""
    import ctypes

    from paper_2601_10729_b200 import _native

    lib = _native.load()
    for b in (1, 3, 16, 64):
        for hq, hkv in ((8, 1), (32, 8), (64, 8), (16, 1), (4, 4)):
            for seq in (0, 1, 15, 16, 17, 1000, 32768, 131072, 1 << 20):
                bps, ns = _split_plan(lib, b, hq, hkv, seq)
                nblk = -(-seq // 16)
                assert 1 <= bps <= 256 and 1 <= ns <= 256
                assert bps * ns >= nblk
                assert ns == max(1, -(-nblk // bps))
    assert _split_plan(lib, 16, 32, 8, 32768) == (256, 8)    # the cfg2 layer: 1024 CTAs
    bad = ctypes.c_int32()
    assert lib.ofb_attention_split_plan(1, 6, 4, 100, 148, 2, ctypes.byref(bad), ctypes.byref(bad)) != 0


def _instep_plan(lib, b, hq, hkv, seq, sms=148, occ=3):
    import ctypes

    bps, ns, narrow = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    assert lib.ofb_attention_instep_plan(b, hq, hkv, seq, sms, occ, ctypes.byref(bps),
                                         ctypes.byref(ns), ctypes.byref(narrow)) == 0
    return bps.value, ns.value, narrow.value


def test_k1_instep_plan_follows_the_sweep():
    """The attention-only in-step K1 plan takes the balanced narrow grid exactly where
    tools/k1_instep_sweep.py measured it > 5 % faster than the cost-model plan, and the
    cost-model plan where that was > 5 % faster (profiles/r02_k1_instep_sweep.jsonl;
    the sequence length in a step is the context + 1)."""
    from paper_2601_10729_b200 import _native

    lib = _native.load()
    heads = {"8B": (32, 8), "70B-TP8-shard": (8, 1)}
    bal_wins = [("8B", 1, 4096), ("8B", 1, 8192), ("8B", 1, 16384), ("8B", 2, 1024),
                ("8B", 2, 4096), ("8B", 2, 8192), ("8B", 4, 1024), ("8B", 4, 4096),
                ("8B", 8, 1024), ("8B", 16, 1024), ("70B-TP8-shard", 2, 65536),
                ("70B-TP8-shard", 4, 32768), ("70B-TP8-shard", 4, 65536),
                ("70B-TP8-shard", 8, 8192), ("70B-TP8-shard", 8, 16384),
                ("70B-TP8-shard", 8, 32768), ("70B-TP8-shard", 16, 4096),
                ("70B-TP8-shard", 16, 8192), ("70B-TP8-shard", 16, 16384)]
    split_wins = ([("70B-TP8-shard", 1, c) for c in (1024, 4096, 8192, 16384, 32768, 65536)]
                  + [("70B-TP8-shard", 2, c) for c in (1024, 4096, 8192, 16384, 32768)]
                  + [("70B-TP8-shard", 4, c) for c in (1024, 4096, 8192, 16384)]
                  + [("70B-TP8-shard", 8, 1024), ("70B-TP8-shard", 8, 4096)])
    for name, b, ctx in bal_wins + split_wins:
        hq, hkv = heads[name]
        bps, ns, narrow = _instep_plan(lib, b, hq, hkv, ctx + 1)
        nblk = -(-(ctx + 1) // 16)
        nominal = max(1, (148 - b * hkv) // (b * hkv))    # one narrow CTA per SM less one per pair
        balanced = narrow == 1 and bps == -(-nblk // nominal) and ns == -(-nblk // bps)
        assert balanced == ((name, b, ctx) in bal_wins), (name, b, ctx, bps, ns, narrow)
        assert ns * bps >= nblk and bps <= 256 and ns <= 256


def test_k1_instep_plan_rejects_bad_shapes():
    import ctypes

    from paper_2601_10729_b200 import _native

    lib = _native.load()
    bad = ctypes.c_int32()
    assert lib.ofb_attention_instep_plan(1, 6, 4, 100, 148, 3, ctypes.byref(bad), ctypes.byref(bad),
                                         ctypes.byref(bad)) != 0
