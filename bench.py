"""Benchmark of the per-decode-step KV data path (BASELINE.json config 2).

Workload (default ``--config cfg2``): Llama-3.1-8B attention shape (32 layers,
32 q / 8 KV heads, d=128, bf16 KV), batch 16, prompts of 32760 tokens
(mid-block), placement ``from_strides(..., [2]*16)``: layers
2,4,..,32 of every request live in pinned host memory (50%), the rest in HBM.
One step = K3 append + K2 fetch of every offloaded slab (32 GiB over PCIe)
+ K1 attention on all 32 layers, enqueued by one native runtime call.

Prints one JSON line (rank 0).  ``value``: tokens/s with step inputs resident
in HBM; ``e2e``: the same through the public API with q / k_new / v_new
copied from pinned host memory and the attention output read back every
step.  ``roofline``: K1 (the dominant kernel) vs measured HBM copy peak;
``step_roofline``: the binding host link (north-star target >= 0.70).
``--impl reference``: the reference has no GPU path and no attention at all
(kvsim prices steps); its arm times the CPU restatement of the data path
(oracle/, kind "port") on this host's cores.
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decode tokens/sec + TPOT SLO attainment; per-step attn+fetch GB/s vs HBM/PCIe roofline"
PCIE5_NOMINAL_GBS = 63.0

CONFIGS = {
    # name: (layers, hq, hkv, batch, prompt, stride, output)
    "cfg1": dict(layers=4, hq=8, hkv=2, batch=4, prompt=4088, strides=[1, 1, None, None],
                 output=64, hidden=1024, workload="toy 4-layer GQA (8q/2kv, d=128), B=4, 4K ctx, reference "
                                     "solve plan: requests 0,1 fully host-resident"),
    "cfg2": dict(layers=32, hq=32, hkv=8, batch=16, prompt=32760, strides=[2] * 16, output=64,
                 hidden=4096,
                 workload="Llama-3.1-8B shape (32 layers, 32q/8kv, d=128, bf16), B=16, 32K ctx, "
                          "stride-2 plan: 50% of layers' KV host-resident, 1xB200"),
    "cfg2r": dict(layers=32, hq=32, hkv=8, batch=16, prompt=32760, strides=[None] * 16, output=64,
                  hidden=4096,
                  workload="Llama-3.1-8B shape, B=16, 32K ctx, every layer HBM-resident "
                           "(pure K1 chain; HBM-bound reference point for cfg2)"),
    "cfg4": dict(layers=80, hq=64, hkv=8, batch=32, prompt=65528, strides="flexgen_plus",
                 output=64, hidden=8192, intermediate=28672,
                 workload="Llama-3.1-70B shape (80 layers, 64q/8kv, d=128, hidden 8192, MLP 28672, "
                          "bf16), B=32, 64K ctx, KV-head sharded TP, whole decoder step (QKV / "
                          "o-proj / MLP weights streamed, o-proj and down-proj all-reduces), plan = "
                          "plan_flexgen_plus under each rank's HBM budget"),
}


def _env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def _probe_link(dev, nbytes: int = 1 << 30, reps: int = 10):
    """Best-of-10 pinned 1 GiB cudaMemcpyAsync H2D / D2H on this GPU."""
    import torch

    from paper_2601_10729_b200 import _native
    from paper_2601_10729_b200.runtime import link_probe

    lib = _native.load()
    host = lib.ofb_host_alloc(nbytes)
    if not host:
        raise RuntimeError("pinned probe buffer allocation failed")
    try:
        d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        return link_probe(host, d.data_ptr(), nbytes, reps)
    finally:
        lib.ofb_host_free(host)


def _standalone_k1(ex, batch, placement, inputs, iters: int = 8):
    """Median CUDA-event time of K1 alone on the first fully resident layer."""
    import numpy as np
    import torch

    from paper_2601_10729_b200 import ops

    ex.drain()
    layer = next((l for l in range(placement.num_layers)
                  if all(row[l] == 1 for row in placement.rows)), None)
    if layer is None:
        return None
    layout = ex._layout(batch)
    host_lens = [r.total_tokens for r in batch]
    max_len = max(host_lens)                      # host-side: no device sync per launch
    lens = torch.tensor(host_lens, dtype=torch.int32, device=ex.device)
    q = inputs["q"][layer]
    out = torch.empty_like(q)
    ws = ex._workspace(len(batch), max_len)
    # back-to-back launches, events in between: the host enqueues far faster than
    # the kernel runs, so intervals after the first are pure device time
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(iters + 2)]
    evs[0].record()
    for i in range(1, iters + 2):
        ops.decode_attention(q, ex.pool.tensor, layout["tables"][layer], lens,
                             max_seq_len=max_len, out=out, ws=ws)
        evs[i].record()
    evs[-1].synchronize()
    times = [evs[i].elapsed_time(evs[i + 1]) for i in range(1, iters + 1)]
    return float(np.median(times))


def _stream_summary(per_stream, nominal_gbs, peak_gbs):
    """Host-link GB/s per copy stream: bytes / the stream's busy time (sum of its
    copies' spans).  The copy engine runs the streams' slab copies essentially one
    at a time at the full link rate, so each stream's rate while busy is the link
    rate and the busy times add up to the step's copy span."""
    rates = [s["bytes"] / (s["busy_ms"] * 1e-3) / 1e9 for s in per_stream if s["busy_ms"] > 0]
    if not rates:
        return None
    return {"streams": len(rates), "GBps_while_busy_min": min(rates),
            "GBps_while_busy_median": statistics.median(rates), "GBps_while_busy_max": max(rates),
            "median_over_h2d_peak": statistics.median(rates) / peak_gbs,
            "median_over_pcie5_nominal": statistics.median(rates) / nominal_gbs,
            "busy_ms_sum": sum(s["busy_ms"] for s in per_stream),
            "bytes_per_stream": [s["bytes"] for s in per_stream][:16]}


def _native_variant(batch, hkv, max_seq_len) -> int:
    from paper_2601_10729_b200 import _native

    return int(_native.load().ofb_attention_variant_for(batch, hkv, max_seq_len))


def _mem_available() -> int:
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 1 << 40


def _measured_peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def _ncu_traffic(alg_bytes):
    """DRAM bytes per K1 launch from the committed ncu --set full capture of the
    same layer shape (profiles/), scaled to this launch's algorithmic bytes."""
    from paper_2601_10729_b200 import ops

    paths = sorted((ROOT / "profiles").glob("*ncu_full_cfg2layer.json"), reverse=True)
    # the capture of the K1 variant that runs at this shape first
    split = bool(_native_variant(16, 8, 32768))
    paths.sort(key=lambda p: (("k1split" in p.name) != split))
    for path in paths:
        try:
            rec = json.loads(path.read_text())[0]
            unit = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
            rd = float(rec["dram__bytes_read.sum"][0]) * unit[rec["dram__bytes_read.sum"][1]]
            wr = float(rec["dram__bytes_write.sum"][0]) * unit[rec["dram__bytes_write.sum"][1]]
            captured_alg = 16 * 32768 * 8 * 2 * 128 * 2 + 2 * 16 * 32 * 128 * 2
            return {"bytes": (rd + wr) * alg_bytes / captured_alg,
                    "ratio_to_algorithmic": (rd + wr) / captured_alg, "source": path.name}
        except Exception:
            continue
    return None


def decoder_weight_bytes(cfg, shard) -> int:
    """Bytes of one rank's weights for the whole-decoder step:
    per layer q/k/v + o rows of its heads, and its 1/TP of gate/up/down."""
    H, inter = cfg["hidden"], cfg["intermediate"] // shard.world
    per_layer = ((shard.local_q + 2 * shard.local_kv) * 128 * H + shard.local_q * 128 * H
                 + 3 * inter * H) * 2
    return cfg["layers"] * per_layer


def build_batch(cfg, shape=None, hbm_budget_bytes=None):
    """Batch + placement.  Fixed stride lists come from the config; "flexgen_plus"
    asks the reference-exact baseline planner (src/policies.py:132-137) for the
    best uniform stride under this rank's HBM budget."""
    from paper_2601_10729_b200.calibrate import b200_profile
    from paper_2601_10729_b200.core import PlacementMatrix, RequestState
    from paper_2601_10729_b200.policies import plan_flexgen_plus

    batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=cfg["prompt"],
                          target_output_tokens=cfg["output"]) for i in range(cfg["batch"])]
    if cfg["strides"] == "flexgen_plus":
        budget = int(hbm_budget_bytes // shape.block_bytes)
        profile = b200_profile(cfg["layers"], shape.num_kv_heads, budget)
        return batch, plan_flexgen_plus(batch, profile)
    placement = PlacementMatrix.from_strides([r.id for r in batch], cfg["layers"], cfg["strides"])
    return batch, placement


class CpuAttentionSample:
    """The CPU restatement of K1 (oracle/attn_oracle.c, all host threads) over
    host-resident KV of one layer per call: the cpu_baseline / reference arm."""

    def __init__(self, shape, batch, arena=None, arena_tables=None):
        import numpy as np

        import oracle

        self.oracle = oracle
        self.threads = oracle.host_threads()
        B = len(batch)
        self.lens = np.array([r.total_tokens + 1 for r in batch], dtype=np.int32)
        nblk = [-(-int(t) // 16) for t in self.lens]
        rng = np.random.default_rng(0)
        if arena is None:
            total = sum(nblk)
            vals = rng.standard_normal(size=total * shape.block_bytes // 2, dtype=np.float32)
            self.pool = (vals.view(np.uint32) >> 16).astype(np.uint16).reshape(
                total, shape.num_kv_heads, 2, 16, 128)
            del vals
            tables = np.full((B, max(nblk)), -1, dtype=np.int32)
            cur = 0
            for b, n in enumerate(nblk):
                tables[b, :n] = np.arange(cur, cur + n)
                cur += n
            self.tables = [tables]
        else:
            self.pool = arena.view_u16(0, arena.blocks).reshape(
                arena.blocks, shape.num_kv_heads, 2, 16, 128)
            self.tables = arena_tables
        self.q = (rng.standard_normal((B, shape.num_q_heads, 128), dtype=np.float32)
                  .view(np.uint32) >> 16).astype(np.uint16)
        self.scale = 1.0 / math.sqrt(128)

    def run(self, seconds_target: float):
        """Attend layer after layer until ~seconds_target; returns (s/layer, layers)."""
        t0 = time.perf_counter()
        done = 0
        while True:
            self.oracle.decode_attention(self.q, self.pool, self.tables[done % len(self.tables)],
                                         self.lens, self.scale, threads=self.threads)
            done += 1
            el = time.perf_counter() - t0
            if el >= seconds_target or done >= 64 or el / done * (done + 1) > seconds_target * 1.5:
                return el / done, done


def reference_control_sample(cfg, decode_tokens: int = 12):
    """The reference's own per-step host control, timed on one core.

    Runs the UNMODIFIED reference ``kvsim`` (imported as its own package from
    ``baseline/_ref``, none of this repo's modules on the path) end to end on the
    config's batch: ``Simulation.execute`` with the reference's baseline planner
    FLEXGEN_PLUS (the policy that yields the config's uniform-stride plan,
    src/policies.py:132-137), i.e. the engine boundary, plan, ``apply_plan`` and
    ``batch_decode_latency_fast`` of every step (src/engine.py:706-734).  Returns
    wall ms per decode step of that Python control loop; kvsim prices steps, so
    this is all the reference executes per step."""
    ref_root = ROOT / "baseline" / "_ref"
    if not (ref_root / "kvsim" / "engine.py").is_file():
        return {"unavailable": "reference kvsim not installed in baseline/_ref"}
    if str(ref_root) not in sys.path:
        sys.path.insert(0, str(ref_root))
    import kvsim

    kvb = cfg["hkv"] * 2 * 128 * 2
    blocks_per_req = -(-(cfg["prompt"] + decode_tokens + 1) // 16)
    # budget: the resident half of the stride-2 plan plus its Eq. 1 buffer
    budget = blocks_per_req * cfg["batch"] * (cfg["layers"] // 2 + 1)
    profile = kvsim.SystemProfile(num_layers=cfg["layers"], compute_base_ms=0.012,
                                  compute_per_token_ms=kvb / 6.4e9,
                                  bandwidth_blocks_per_ms=55.6e6 / (kvb * 16),
                                  gpu_block_budget=budget, block_size=16)
    slo = kvsim.SloConfig(tbt_target_ms=1000.0, tpot_target_ms=1000.0)
    trace = kvsim.Trace(tuple(kvsim.TraceRequest(0, cfg["prompt"], decode_tokens)
                              for _ in range(cfg["batch"])))
    run_cfg = kvsim.RunConfig(max_batch=cfg["batch"], batch_token_cap=1 << 40)
    policy = kvsim.make_policy(kvsim.PolicyKind.FLEXGEN_PLUS, profile, slo, None,
                               max_batch=run_cfg.max_batch, token_cap=run_cfg.batch_token_cap)
    t0 = time.perf_counter()
    log = kvsim.Simulation(trace, policy, profile, slo, run_cfg).execute()
    wall = time.perf_counter() - t0
    steps = [r for r in log if r["kind"] == "step"]
    offl = sum(1 for row in steps[-1]["payload"]["rows"] for x in row if x == 0)
    return {"ms_per_step": wall * 1e3 / max(1, len(steps)), "steps": len(steps),
            "cores": 1, "cores_of": len(os.sched_getaffinity(0)),
            "policy": "flexgen_plus", "offloaded_slabs_last_step": offl,
            "module": str(Path(kvsim.__file__).parent.relative_to(ROOT)),
            "what": "reference kvsim Simulation.execute wall time / decode steps (engine "
                    "boundary + plan + apply_plan + batch_decode_latency_fast), 1 core"}


def host_dram_gbs(threads: int) -> float:
    """Host DRAM copy bandwidth (SURVEY.md 8(d) CPU baseline item 2): best of 5
    torch CPU copies of 1 GiB on `threads` threads, read + write bytes / time -
    the same method as the HBM copy peak."""
    import torch

    prev = torch.get_num_threads()
    torch.set_num_threads(threads)
    try:
        src = torch.empty(1 << 30, dtype=torch.uint8).fill_(1)
        dst = torch.empty_like(src)
        best = float("inf")
        for _ in range(5):
            t0 = time.perf_counter()
            dst.copy_(src)
            best = min(best, time.perf_counter() - t0)
        return 2 * src.numel() / best / 1e9
    finally:
        torch.set_num_threads(prev)


def run_reference_arm(args, cfg):
    """The reference path on this host: kvsim's own control loop (1 core) plus
    the CPU restatement of the data path it prices (oracle port: K3 append + K1
    attention of every layer, all host threads), timed as WHOLE steps."""
    from paper_2601_10729_b200.executor import ModelShape

    import numpy as np

    import oracle

    rank, world, _ = _env_rank()
    if rank != 0:
        return
    shape = ModelShape(cfg["layers"], cfg["hq"], cfg["hkv"])
    # the CPU arm attends every layer of host-resident KV: no placement needed
    batch, _placement = build_batch(dict(cfg, strides=[None] * cfg["batch"]))
    sampler = CpuAttentionSample(shape, batch)
    threads = sampler.threads
    B = len(batch)
    rng = np.random.default_rng(1)
    knew = (rng.standard_normal((B, shape.num_kv_heads, 128), dtype=np.float32)
            .view(np.uint32) >> 16).astype(np.uint16)
    vnew = knew[::-1].copy()
    pos = sampler.lens - 1

    def whole_step():
        # one pool stands in for every layer's slabs (68 GB of distinct KV would not
        # fit host RAM at cfg2); each layer's 2.1 GB read still misses the LLC
        for _ in range(cfg["layers"]):
            oracle.kv_append(knew, vnew, sampler.pool, sampler.tables[0], pos)
            oracle.decode_attention(sampler.q, sampler.pool, sampler.tables[0], sampler.lens,
                                    sampler.scale, threads=threads)

    control = reference_control_sample(cfg)
    ctl_ms = control.get("ms_per_step", 0.0)
    for _ in range(args.warmup):
        whole_step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        whole_step()
        times.append(time.perf_counter() - t0)
    data_ms = statistics.median(times) * 1e3
    step_ms = data_ms + ctl_ms
    value = cfg["batch"] / (step_ms * 1e-3)
    kv_bytes = int(sum(int(t) for t in sampler.lens)) * cfg["hkv"] * 2 * 128 * 2
    cpu_gbs = kv_bytes * cfg["layers"] / (data_ms * 1e-3) / 1e9
    dram_gbs = host_dram_gbs(threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64-accum over bf16 KV", "data": "synthetic",
        "config": {"workload": cfg["workload"],
                   "sample": f"whole {cfg['layers']}-layer steps of {cfg['batch']} requests, "
                             "timed unscaled"},
        "step_ms": {"data_path_median": data_ms, "control": ctl_ms,
                    "data_path_all": [t * 1e3 for t in times]},
        "cpu_gbs": cpu_gbs,
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "port",
                         "kv_read_gbs": cpu_gbs, "host_dram_copy_gbs": dram_gbs,
                         "frac_of_host_dram": cpu_gbs / dram_gbs,
                         "sample": f"whole steps: {cfg['layers']} layers x (append + attention "
                                   f"of {cfg['batch']} requests x {cfg['prompt']} tokens), "
                                   "oracle/attn_oracle.c accumulating in f64 over bf16 KV "
                                   f"on {threads} threads, + the reference kvsim control loop "
                                   "on 1 core (kvsim has no attention of its own)",
                         "control": control},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, cfg):
    import numpy as np
    import torch

    from paper_2601_10729_b200 import ops
    from paper_2601_10729_b200.executor import B200Executor, ModelShape
    from paper_2601_10729_b200.latency import blocks_to_fetch
    from paper_2601_10729_b200.runtime import link_probe

    rank, world, local = _env_rank()
    # one rank per GPU; OFB_DIST_BACKEND=gloo + several ranks per GPU is only for
    # exercising the multi-rank path on a single-GPU box (tests), never for numbers
    local = local % max(1, torch.cuda.device_count())
    dist = None
    if world > 1:
        import torch.distributed as dist  # noqa: F811

        torch.cuda.set_device(local)
        dist.init_process_group(os.environ.get("OFB_DIST_BACKEND", "nccl"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    from paper_2601_10729_b200.tp import HeadShard, TensorParallelDecoder

    hkv_total, hq_total = cfg["hkv"], cfg["hq"]
    tp = world if world > 1 else max(1, args.tp_emulate)
    if hkv_total % tp:
        raise SystemExit(f"KV heads ({hkv_total}) must divide by the TP degree ({tp})")
    # KV-head sharding: each rank owns Hkv/N KV heads + their q heads
    shard = HeadShard(rank if world > 1 else 0, tp, hq_total, hkv_total)
    shape = ModelShape(cfg["layers"], shard.local_q, shard.local_kv)
    L, B = cfg["layers"], cfg["batch"]
    # every request must have tokens left for all the steps this run makes
    # (warm-up, timed, instrumented, e2e warm-up + timed)
    cfg = dict(cfg, output=max(cfg["output"], args.warmup + 2 * args.steps + 3 + 8 + 16))
    cap = -(-(cfg["prompt"] + cfg["output"] + 1) // 16)
    slots = args.staging_slots
    use_tp = world > 1 or args.tp_emulate > 1 or cfg["strides"] == "flexgen_plus"
    full = (args.decoder or ("full" if "intermediate" in cfg else "attn")) == "full"
    if full and "intermediate" not in cfg:
        raise SystemExit(f"--decoder full needs an MLP shape; {args.config} is attention-only")
    # per-rank HBM left for KV: total - weights (o-proj shard, or the whole decoder
    # shard) - staging - workspace/slack
    free_b, _total_b = torch.cuda.mem_get_info(dev)
    oproj_bytes = (decoder_weight_bytes(cfg, shard) if full else
                   L * shard.local_q * 128 * cfg["hidden"] * 2 if use_tp else 0)
    staging_bytes = B * slots * cap * shape.block_bytes
    kv_budget = free_b - oproj_bytes - staging_bytes - (6 << 30)
    if dist is not None:
        # C2: every rank must plan with the same budget - the smallest
        t = torch.tensor([kv_budget], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        kv_budget = int(t.item())
    batch, placement = build_batch(cfg, shape, kv_budget)
    if dist is not None:
        from paper_2601_10729_b200.tp import check_plan_replicated

        if not check_plan_replicated(placement.rows):
            raise SystemExit("ranks computed different placements (C2 violated)")
    n_off = sum(row.count(0) for row in placement.rows)
    n_res = L * B - n_off
    host_need = n_off * cap * shape.block_bytes
    avail = _mem_available() // max(1, world)
    if host_need > 0.85 * avail:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "config": {"workload": cfg["workload"]},
                              "n_gpus": world, "tp": tp, "unavailable":
                              f"needs {host_need / 2**30:.0f} GiB pinned host KV per rank, "
                              f"{avail / 2**30:.0f} GiB available"}), flush=True)
        return
    device_blocks = n_res * cap + B * slots * cap + 16
    host_blocks = max(n_off * cap, 1) + 16
    ex = B200Executor(shape, device=dev, device_blocks=device_blocks, host_blocks=host_blocks,
                      staging_slots=slots, copy_streams=args.copy_streams, seed=rank,
                      record_timing=True)
    # host-link peaks on this GPU (1 GiB pinned, best of 10) - before the data lands
    h2d_peak, d2h_peak = _probe_link(dev)
    ex.install(batch, placement)
    torch.cuda.synchronize()

    inputs = [ex.synthetic_inputs(B, step=i) for i in range(2)]
    attn_tokens = []

    if full:
        from paper_2601_10729_b200.tp import TensorParallelLlama

        # whole decoder: the step's input is the new tokens' embeddings, its result
        # the last hidden state; q / k_new / v_new come from the QKV projections
        tpd = TensorParallelLlama(ex, shard, cfg["hidden"], cfg["intermediate"], c1=args.c1,
                                  seed=0, max_batch=B)
        g = torch.Generator(device=dev)
        g.manual_seed(17)
        step_in = [{"x": torch.randn((B, cfg["hidden"]), generator=g, device=dev).to(torch.bfloat16)}
                   for _ in range(2)]
        result = lambda: tpd.last_hidden  # noqa: E731
    else:
        tpd = TensorParallelDecoder(ex, shard, cfg["hidden"], seed=0, max_batch=B) if use_tp else None
        step_in = inputs
        result = lambda: ex.last_output  # noqa: E731
    pinned = [{k: v.cpu().pin_memory() for k, v in inp.items()} for inp in step_in]
    out_host = (torch.empty((B, cfg["hidden"]), dtype=torch.bfloat16) if full
                else torch.empty_like(inputs[0]["q"], device="cpu")).pin_memory()

    def run_step(inp):
        if full:
            tpd.step(batch, inp["x"])
        elif tpd is not None:
            tpd.step(batch, inp)
        else:
            ex.decode_step(batch, None, inp, sync=False)

    def step(i, e2e=False):
        attn_tokens.append(sum(r.total_tokens + 1 for r in batch))
        if e2e:   # a serving loop: inputs from host, result read back before the next step
            dev_in = {k: v.to(dev, non_blocking=True) for k, v in pinned[i % 2].items()}
            run_step(dev_in)
            out_host.copy_(result(), non_blocking=True)
            torch.cuda.current_stream().synchronize()
        else:     # device-resident inputs, steps pipelined (host prepares N+1 during N)
            run_step(step_in[i % 2])
        for r in batch:
            r.record_generated_token()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def clean_boundary():
        """No cross-step prefetch crosses a timing boundary: nothing is in flight
        when a timed region starts (the first step fetches everything itself) and
        the last step of a region issues none, so a region holds exactly its own
        steps' transfers."""
        ex.drain()
        ex.runtime.prefetch_fence()
        barrier()

    def run_steps(n, e2e=False, marks=None):
        for i in range(n):
            ex.prefetch_next = i < n - 1
            step(i, e2e=e2e)
            if marks is not None:
                marks.append(time.perf_counter())
        ex.prefetch_next = True

    for i in range(args.warmup):
        step(i)
    clean_boundary()
    # --layer-events inline (default): per-launch K1 / per-copy events inside the
    # timed steps.  separate: the timed steps carry none (an event between two
    # kernels breaks their programmatic-dependent-launch overlap) and per-launch K1
    # times and per-copy bytes come from a separate instrumented pass below.
    inline = args.layer_events == "inline"
    ex.record_timing = inline
    ex.runtime.timing_reset()
    attn_tokens.clear()
    with ClockSampler(local) as clocks:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record()
        run_steps(args.steps)
        t_end.record()
        ex.drain()
        barrier()
    total_ms = t_start.elapsed_time(t_end)
    if not inline:
        clean_boundary()
        ex.record_timing = True
        ex.runtime.timing_reset()
        attn_tokens.clear()
        run_steps(min(args.steps, 3))
        ex.drain()
        barrier()
    tm = ex.runtime.timing()   # per-launch K1 events + fetch bytes of the instrumented steps
    per_stream = ex.runtime.stream_stats()
    k1_tokens = list(attn_tokens)
    ex.record_timing = False   # e2e: a serving loop, no instrumentation
    if dist is not None:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps

    # e2e through the public API with host buffers (untimed warm-up steps first:
    # the caching allocator settles the per-step input / output tensors)
    for i in range(3):
        step(i, e2e=True)
    clean_boundary()
    pf0 = ex.runtime.prefetch_stats()
    gc_pauses = []          # interpreter GC pauses inside the e2e region (host outliers)
    gc_t0 = [0.0]

    def _gc_cb(phase, info):
        if phase == "start":
            gc_t0[0] = time.perf_counter()
        else:
            gc_pauses.append((info.get("generation"), round((time.perf_counter() - gc_t0[0]) * 1e3, 3)))
    gc.callbacks.append(_gc_cb)
    e0 = time.perf_counter()
    e2e_steps = max(8, args.steps)
    marks = [e0]
    run_steps(e2e_steps, e2e=True, marks=marks)
    barrier()
    gc.callbacks.remove(_gc_cb)
    e2e_step_ms = [(b - a) * 1e3 for a, b in zip(marks, marks[1:])]
    pf1 = ex.runtime.prefetch_stats()
    e2e_ms = (time.perf_counter() - e0) * 1e3 / e2e_steps
    if dist is not None:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    # K1 alone on one resident layer of the same state (no concurrent DMA), to
    # separate the kernel's own efficiency from in-step link interference
    standalone = _standalone_k1(ex, batch, placement, inputs[0])
    h2d_in = sum(v.numel() * v.element_size() for v in pinned[0].values())
    d2h_out = out_host.numel() * out_host.element_size()

    # roofline of K1 (dominant kernel): algorithmic bytes per launch / event duration
    peaks = _measured_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    attn_ms = tm["acc_attn_ms"] / tm["acc_attn_launches"]
    tokens_per_layer = sum(k1_tokens) / len(k1_tokens)
    kv_bytes = tokens_per_layer * shape.kv_bytes_per_token
    qo_bytes = 2 * B * shape.num_q_heads * 128 * 2
    attn_bytes = kv_bytes + qo_bytes
    attn_gbs = attn_bytes / (attn_ms * 1e-3) / 1e9

    # step roofline: host link (HOST_alg) vs HBM (HBM_alg), SURVEY.md 8(d)
    host_alg = tm["acc_copy_bytes"] / tm["acc_steps"]
    weight_bytes = tpd.weight_bytes if full else 0
    hbm_alg = L * attn_bytes + B * L * shape.kv_bytes_per_token + weight_bytes
    roof_ms = max(hbm_alg / (hbm_peak * 1e9), host_alg / (h2d_peak * 1e9)) * 1e3
    copy_span = tm["copy_span_ms"]
    bound = "host_link" if host_alg / h2d_peak > hbm_alg / hbm_peak else "hbm"

    traffic = _ncu_traffic(attn_bytes)
    value = B / (ms_per_step * 1e-3)  # whole job: every rank serves the same B tokens (TP)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        off_layers = sorted({l for row in placement.rows for l, bit in enumerate(row) if bit == 0})
        tables = []
        for l in off_layers[:4]:
            if any(ex.slabs[r.id].host[l] is None for r in batch):
                continue
            t = np.full((B, cap), -1, dtype=np.int32)
            for b, r in enumerate(batch):
                t[b] = ex.slabs[r.id].host[l] + np.arange(cap, dtype=np.int32)
            tables.append(t)
        sampler = CpuAttentionSample(shape, batch, arena=ex.host, arena_tables=tables) \
            if tables else CpuAttentionSample(shape, batch)
        per_layer_s, layers_done = sampler.run(args.ref_seconds)
        cpu_step = per_layer_s * L
        cpu = {"value": B / cpu_step, "unit": "tokens/s", "cores": sampler.threads, "kind": "port",
               "sample": f"{layers_done} layer(s) x {B} requests x ~{cfg['prompt']} tokens of "
                         f"host-resident KV through oracle/attn_oracle.c, scaled to {L} layers"}
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded N(0,1) KV, q)",
        "config": {"workload": cfg["workload"], "global_batch": B, "seq_len": cfg["prompt"],
                   "layers": L, "q_heads": hq_total, "kv_heads": hkv_total,
                   "parallelism": (f"tp{world} (KV-head sharded; C1 per layer: "
                                   + ("K6, tcgen05 projection fused with a one-shot all-reduce over "
                                      "NVLink peer memory)" if args.c1 == "k6" else
                                      "cuBLAS projection + NCCL all-reduce)")
                                   if world > 1 else
                                   f"tp{tp} rank-0 shard emulated on 1 GPU ({args.c1} projections, "
                                   "no exchange)" if tp > 1 else "single GPU"),
                   "decoder": ("whole Llama layer per step: RMSNorm, QKV / gate-up (cuBLAS), K3+K1, "
                               f"o-proj + down-proj with all-reduce ({args.c1}); "
                               f"{weight_bytes / 1e9:.2f} GB of weights streamed per step"
                               if full else "attention path (K3 + K2 + K1" +
                               (" + K6 o-proj)" if tpd is not None else ")")),
                   "placement_rows_offloaded": [row.count(0) for row in placement.rows][:4],
                   "offloaded_slabs": n_off, "staging_slots": slots,
                   "copy_streams": tm["copy_streams"], "host_pipelining": "4 steps in flight",
                   "k1_timing": ("CUDA events around every K1 launch inside the timed steps"
                                 if inline else "CUDA events in a separate instrumented pass of "
                                 f"{len(k1_tokens)} steps (timed steps carry no per-layer events)"),
                   "l2": "inputs (64 GiB KV) larger than the 126 MB L2; no flush needed"},
        "e2e": {"value": B / (e2e_ms * 1e-3), "unit": "tokens/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": h2d_in, "d2h_bytes_per_step": d2h_out,
                "step_ms": [round(x, 3) for x in e2e_step_ms],
                "gc_pauses": [{"gen": g_, "ms": m_} for g_, m_ in gc_pauses if m_ >= 0.5],
                "prefetch_adopted_steps": pf1["adopted"] - pf0["adopted"],
                "prefetch_dropped_steps": pf1["dropped"] - pf0["dropped"]},
        "roofline": {"bound": "hbm", "kernel": ("K1 paged GQA decode (" + ("paged_gqa_decode_kernel, split variant"
                                  if _native_variant(B, shape.num_kv_heads, int(tokens_per_layer / B))
                                  else "paged_gqa_decode_stream_kernel, stream-K variant") + ")"),
                     "achieved": attn_gbs, "peak": hbm_peak, "unit": "GB/s",
                     "frac": attn_gbs / hbm_peak,
                     "traffic": (traffic or {}).get("bytes"),
                     "traffic_over_algorithmic": (traffic or {}).get("ratio_to_algorithmic"),
                     "traffic_source": (traffic or {}).get("source"),
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)",
                     "bytes_per_launch": attn_bytes, "launch_ms": attn_ms,
                     "frac_of_8tbs_nominal": attn_gbs / 8000.0,
                     "standalone": None if standalone is None else {
                         "launch_ms": standalone, "achieved": attn_bytes / (standalone * 1e-3) / 1e9,
                         "frac": attn_bytes / (standalone * 1e-3) / 1e9 / hbm_peak,
                         "note": "same layer, K1 alone: no concurrent fetch DMA into HBM"}},
        "step_roofline": {"bound": bound, "achieved_frac": roof_ms / ms_per_step,
                          "roofline_ms": roof_ms, "measured_ms": ms_per_step,
                          "host_alg_bytes": host_alg, "hbm_alg_bytes": hbm_alg,
                          "h2d_peak_gbs": h2d_peak, "d2h_peak_gbs": d2h_peak,
                          "host_link_gbs": host_alg / (ms_per_step * 1e-3) / 1e9,
                          "copy_span_ms": copy_span,
                          "copy_gbs_during_span": (host_alg / (copy_span * 1e-3) / 1e9
                                                   if copy_span else None),
                          "frac_of_pcie5_nominal": host_alg / (ms_per_step * 1e-3) / 1e9
                          / PCIE5_NOMINAL_GBS,
                          "blocks_to_fetch_check": blocks_to_fetch(placement, batch),
                          "per_copy_stream": _stream_summary(per_stream, PCIE5_NOMINAL_GBS, h2d_peak)},
        "attn_share_of_step": tm["acc_attn_ms"] / max(tm["acc_step_ms"], 1e-9),
        "gpu_launches": args.steps * ((L + L + (2 * L if args.c1 == "k6" else 0)) if full else
                                      (1 + L + len({l for row in placement.rows
                                                    for l, b in enumerate(row) if b == 0})
                                       + (L if tpd is not None else 0))),
        "clocks": clocks.summary(),
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line), flush=True)
    if tpd is not None:
        tpd.close()
    ex.close()
    if dist is not None:
        dist.destroy_process_group()


def run_reconfig(args):
    """Config 5: plan change stride 2 <-> stride 4 on the 8B shape, sweep B x T.

    Each point installs stride 2, decodes, switches to stride 4 (H2D restore of
    the layers = 2 mod 4: reconfiguration_delta = (8*b_r, 0) per request) and back
    (D2H eviction of the same layers), decoding one step after each switch.
    Migration GB/s per direction is measured with CUDA events on the runtime's
    migration streams; the reference only charges h2d_blocks / bandwidth
    (src/engine.py:248) and treats D2H as free.
    """
    import torch

    from paper_2601_10729_b200.core import PlacementMatrix, RequestState
    from paper_2601_10729_b200.executor import B200Executor, LLAMA31_8B
    from paper_2601_10729_b200.latency import reconfiguration_delta
    from paper_2601_10729_b200.runtime import link_probe

    shape = LLAMA31_8B
    max_tokens = args.sweep_max_tokens
    points = [(b, t) for b in (1, 2, 4, 8, 16, 32, 64) for t in (16384, 32768, 65536, 131072)
              if b * t <= max_tokens]
    cap_of = lambda t: -(-(t + 64 + 1) // 16)  # noqa: E731
    dev_blocks = max(int(0.75 * b * shape.num_layers * cap_of(t)) + b * cap_of(t) for b, t in points) + 64
    host_blocks = max(b * (shape.num_layers // 2) * cap_of(t) for b, t in points) + 64
    ex = B200Executor(shape, device_blocks=dev_blocks, host_blocks=host_blocks, record_timing=True,
                      fill="zeros")
    h2d_peak, d2h_peak = _probe_link(ex.device)
    results = []
    for b, t in points:
        batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=t - 8, target_output_tokens=64)
                 for i in range(b)]
        ids = [r.id for r in batch]
        s2 = PlacementMatrix.from_strides(ids, shape.num_layers, [2] * b)
        s4 = PlacementMatrix.from_strides(ids, shape.num_layers, [4] * b)
        ex.install(batch, s2)
        base_ms = ex.decode_step(batch, s2)
        rec = {"batch": b, "context": t}
        for name, old, new in (("restore_h2d", s2, s4), ("evict_d2h", s4, s2)):
            up, down = reconfiguration_delta(old, new, batch)
            ex.install(batch, new)
            tm = ex.runtime.timing()
            step_ms = ex.decode_step(batch, new)
            nbytes = tm["mig_h2d_bytes"] + tm["mig_d2h_bytes"]
            rec[name] = {"delta_blocks": [up, down], "bytes": nbytes, "ms": tm["mig_ms"],
                         "GBps": nbytes / (tm["mig_ms"] * 1e-3) / 1e9 if tm["mig_ms"] else None,
                         "frac_of_link_peak": (nbytes / (tm["mig_ms"] * 1e-3) / 1e9)
                         / (h2d_peak if up else d2h_peak) if tm["mig_ms"] else None,
                         "model_charge_ms": up * shape.block_bytes / (h2d_peak * 1e6),
                         "next_step_ms": step_ms}
        rec["step_ms_stride2"] = base_ms
        results.append(rec)
        for r in batch:
            ex.release(r.id)
        torch.cuda.synchronize()
    line = {"metric": "plan-change migration GB/s per direction (config 5)", "config": "cfg5",
            "h2d_peak_gbs": h2d_peak, "d2h_peak_gbs": d2h_peak, "points": results}
    print(json.dumps(line), flush=True)
    ex.close()


def cfg3_setup(args):
    """Config 3: 8B shape, mixed 8K-128K trace, OrbitPolicy with online refinement
    and fallback deferral, B200-calibrated profile."""
    from paper_2601_10729_b200 import defaults, workload
    from paper_2601_10729_b200.calibrate import b200_profile
    from paper_2601_10729_b200.engine import RunConfig

    spec = workload.LengthSpec(kind="lognormal", prompt_median=32768, prompt_sigma=0.6,
                               output_median=args.cfg3_output_median, output_sigma=0.5,
                               max_prompt=131072, max_output=4 * args.cfg3_output_median)
    raw = workload.generate(seed=3, rate=args.cfg3_rate, cv=1.5, length_spec=spec,
                            count=args.cfg3_requests)
    # builder-side min-8K filter
    trace = workload.Trace(tuple(workload.TraceRequest(r.arrival_ms, max(r.prompt_tokens, 8192),
                                                       r.output_tokens) for r in raw.requests),
                           dict(raw.metadata, min_prompt="8192"))
    if args.cfg3_calibrate:   # price with this box's measured K1 / link
        from paper_2601_10729_b200.calibrate import measure_b200_profile

        profile, _raw = measure_b200_profile(32, 32, 8, args.cfg3_budget_blocks)
    else:
        profile = b200_profile(32, 8, gpu_block_budget=args.cfg3_budget_blocks)
    slo = defaults.default_slo(profile, scale=args.slo_scale)
    cfg = RunConfig(max_batch=4, batch_token_cap=600000)
    return trace, profile, slo, cfg


def run_cfg3_policies(args):
    """Config 3 trace under every policy the reference ships (src/policies.py:270-276),
    each on the B200 executor in live mode (measured step time drives the clock):
    the paper's policy comparison (TPOT / TBT attainment, throughput) on real steps."""
    import torch

    from paper_2601_10729_b200.engine import Simulation
    from paper_2601_10729_b200.executor import B200Executor, LLAMA31_8B
    from paper_2601_10729_b200.metrics import collect_metrics
    from paper_2601_10729_b200.policies import PolicyKind, make_policy

    trace, profile, slo, cfg = cfg3_setup(args)
    rows = {}
    wanted = [k.strip() for k in args.cfg3_policies.split(",")] if args.cfg3_policies else None
    for kind in PolicyKind:
        if wanted and kind.value not in wanted:
            continue
        policy = make_policy(kind, profile, slo, max_batch=cfg.max_batch, token_cap=cfg.batch_token_cap)
        ex = B200Executor.for_trace(trace, profile, shape=LLAMA31_8B, max_batch=cfg.max_batch)
        t0 = time.perf_counter()
        try:
            log = Simulation(trace, policy, profile, slo, cfg, executor=ex, mode="live").execute()
        except Exception as exc:   # a policy the budget cannot serve: report, do not hide
            rows[kind.value] = {"error": repr(exc)}
            print(json.dumps({"policy": kind.value, **rows[kind.value]}), file=sys.stderr, flush=True)
            ex.close()
            continue
        wall = time.perf_counter() - t0
        steps = [r for r in log if r["kind"] == "step"]
        gpu_ms = sum(r["payload"]["measured_us"] for r in steps) / 1e3
        tokens = sum(len(r["payload"]["ids"]) for r in steps)
        rep = collect_metrics(log)
        rows[kind.value] = {"steps": len(steps), "tokens": tokens, "gpu_ms": gpu_ms,
                            "tokens_per_s_gpu": tokens / (gpu_ms * 1e-3) if gpu_ms else None,
                            "makespan_ms": max((r["time_us"] for r in log), default=0) / 1e3,
                            "throughput_rpm": rep.throughput_rpm, "tpot_p95_ms": rep.tpot_p95_ms,
                            "tpot_attainment": rep.tpot_attainment,
                            "tbt_attainment": rep.tbt_attainment, "tbt_p95_ms": rep.tbt_p95_ms,
                            "pauses": rep.pauses, "replans": rep.replans,
                            "preemptions": rep.preemptions,
                            "h2d_migrated_bytes": ex.migrated["h2d_bytes"], "wall_s": wall}
        ex.close()
        torch.cuda.synchronize()
        print(json.dumps({"policy": kind.value, **rows[kind.value]}), file=sys.stderr, flush=True)
    print(json.dumps({"metric": METRIC, "config": "cfg3-policies", "mode": "live",
                      "requests": len(trace.requests), "budget_blocks": profile.gpu_block_budget,
                      "policies": rows}), flush=True)


def _recording_executor(base_cls):
    """The executor with per-step algorithmic bytes recorded:
    HOST = blocks_to_fetch x block bytes (src/latency.py:99-105), HBM = the
    resident layers' KV of every request + q / out + the appended token."""
    from paper_2601_10729_b200.latency import blocks_to_fetch

    class Recording(base_cls):
        def decode_step(self, batch, placement=None, inputs=None, sync=True):
            ms = super().decode_step(batch, placement, inputs, sync=sync)
            shape = self.shape
            host = blocks_to_fetch(placement, batch) * shape.block_bytes
            hbm = sum(row.count(1) * (r.total_tokens + 1) for r, row in zip(batch, placement.rows)) \
                * shape.kv_bytes_per_token
            hbm += len(batch) * shape.num_layers * (2 * shape.num_q_heads * 128 * 2
                                                     + shape.kv_bytes_per_token)
            self.step_bytes.append((len(batch), host, hbm))
            return ms

    return Recording


def run_cfg3(args):
    """Config 3 through the serving engine in all three clock modes, side by side:
    parity (model time; decisions must equal the executor-less run), live (the
    measured device step drives the clock) and live-wall (host wall time: solve,
    install, Python and the device step).  Per mode: tokens/s, TPOT / TBT
    attainment, the batch-size histogram, per-step HOST / HBM algorithmic bytes
    against the binding roofline, and host-control ms per step."""
    import torch

    from paper_2601_10729_b200.engine import Simulation
    from paper_2601_10729_b200.executor import B200Executor, LLAMA31_8B
    from paper_2601_10729_b200.metrics import collect_metrics
    from paper_2601_10729_b200.policies import PolicyKind, make_policy

    trace, profile, slo, cfg = cfg3_setup(args)
    peaks = _measured_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6450.0))
    h2d_peak, _d2h = _probe_link(torch.device("cuda"))

    def simulate(executor, mode):
        policy = make_policy(PolicyKind.ORBIT, profile, slo, max_batch=cfg.max_batch,
                             token_cap=cfg.batch_token_cap)
        sim = Simulation(trace, policy, profile, slo, cfg, executor=executor, mode=mode)
        t0 = time.perf_counter()
        log = sim.execute()
        return log, time.perf_counter() - t0

    model_log, model_s = simulate(None, "parity")
    out = {"metric": METRIC, "config": "cfg3",
           "workload": f"Llama-3.1-8B shape, mixed 8K-128K lognormal trace (seed 3, {args.cfg3_rate:g} "
                       "req/s), OrbitPolicy, "
                       f"max_batch 4, HBM budget {profile.gpu_block_budget} blocks x 64 KiB "
                       f"({profile.gpu_block_budget * 65536 / 2**30:.1f} GiB)",
           "requests": len(trace.requests),
           "prompts": [r.prompt_tokens for r in trace.requests],
           "profile": {"source": "measured on this GPU" if args.cfg3_calibrate
                       else "round-1 B200 constants (calibrate.py)",
                       "compute_base_ms": profile.compute_base_ms,
                       "compute_per_token_ms": profile.compute_per_token_ms,
                       "bandwidth_blocks_per_ms": profile.bandwidth_blocks_per_ms},
           "peaks": {"hbm_gbs": hbm_peak, "h2d_gbs": h2d_peak}}
    steps_model = [r for r in model_log if r["kind"] == "step"]
    out["model_host_control_ms_per_step"] = model_s * 1e3 / max(1, len(steps_model))
    recording = _recording_executor(B200Executor)
    for mode in ("parity", "live", "live-wall"):
        ex = recording.for_trace(trace, profile, shape=LLAMA31_8B, max_batch=cfg.max_batch)
        ex.step_bytes = []
        with ClockSampler(0) as clocks:
            log, wall_s = simulate(ex, mode)
        steps = [r for r in log if r["kind"] == "step"]
        gpu = [r["payload"]["measured_us"] / 1e3 for r in steps]
        gpu_ms = sum(gpu)
        tokens = sum(len(r["payload"]["ids"]) for r in steps)
        rep = collect_metrics(log)
        hist = {}
        for b, _h, _m in ex.step_bytes:
            hist[b] = hist.get(b, 0) + 1
        roof = [max(m / (hbm_peak * 1e9), h / (h2d_peak * 1e9)) * 1e3 for _b, h, m in ex.step_bytes]
        link_bound = sum(1 for _b, h, m in ex.step_bytes if h / h2d_peak > m / hbm_peak)
        host = sum(h for _b, h, _m in ex.step_bytes)
        hbm = sum(m for _b, _h, m in ex.step_bytes)
        rec = {"steps": len(steps), "tokens": tokens, "gpu_ms": gpu_ms,
               "tokens_per_s_gpu": tokens / (gpu_ms * 1e-3), "wall_s": wall_s,
               "tpot_attainment": rep.tpot_attainment, "tbt_attainment": rep.tbt_attainment,
               "tpot_p95_ms": rep.tpot_p95_ms, "tbt_p95_ms": rep.tbt_p95_ms,
               "batch_histogram": dict(sorted(hist.items())),
               "mean_batch": tokens / max(1, len(steps)),
               "pauses": rep.pauses, "resumes": rep.resumes, "replans": rep.replans,
               "preemptions": rep.preemptions, "migrated": dict(ex.migrated),
               "prefetch": ex.runtime.prefetch_stats(),
               "step_roofline": {
                   "host_alg_bytes_total": host, "hbm_alg_bytes_total": hbm,
                   "host_link_bound_steps": link_bound, "hbm_bound_steps": len(roof) - link_bound,
                   "host_gbs_over_gpu_time": host / (gpu_ms * 1e-3) / 1e9,
                   "hbm_gbs_over_gpu_time": hbm / (gpu_ms * 1e-3) / 1e9,
                   "roofline_ms_total": sum(roof), "measured_ms_total": gpu_ms,
                   "achieved_frac": sum(roof) / gpu_ms if gpu_ms else None,
                   "per_step_first8": [{"B": b, "host_bytes": h, "hbm_bytes": m,
                                        "roofline_ms": rf, "measured_ms": g}
                                       for (b, h, m), rf, g in list(zip(ex.step_bytes, roof, gpu))[:8]]},
               "clocks": clocks.summary()}
        if mode == "live-wall":
            walls = [r["payload"]["wall_us"] / 1e3 for r in steps if "wall_us" in r["payload"]]
            rec["host_control_ms_per_step_median"] = statistics.median(
                w - g for w, g in zip(walls, gpu)) if walls else None
            rec["tokens_per_s_clock"] = tokens / (sum(walls) * 1e-3) if walls else None
        if mode == "parity":
            stripped = [dict(r, payload={k: v for k, v in r["payload"].items() if k != "measured_us"})
                        if r["kind"] == "step" else r for r in log]
            rec["decisions_match_model_run"] = stripped == model_log
            rec["model_tpot_attainment"] = collect_metrics(model_log).tpot_attainment
        out[mode] = rec
        print(json.dumps({"mode": mode, **{k: v for k, v in rec.items()
                                            if k not in ("step_roofline",)}}), file=sys.stderr, flush=True)
        ex.close()
        torch.cuda.synchronize()
    print(json.dumps(out), flush=True)


def run_cfg4_serve(args):
    """Config 4 through the serving engine: ``engine.Simulation`` drives one
    KV-head-sharded rank per GPU (``tp.TensorParallelExecutor`` over the whole
    decoder step, ``tp.TensorParallelLlama``), plans replicated on every rank
    (C2).  Reports tokens/s, TPOT / TBT attainment and the binding roofline per
    TP degree, in parity mode (decisions must equal the executor-less model run,
    src/engine.py:706-734) and on the live-wall clock (solve + install + Python +
    device step advance the clock).  Under torchrun every rank
    runs the engine; alone, ``--tp-emulate N`` serves rank 0's shard of TP-N."""
    import torch

    from paper_2601_10729_b200 import defaults, workload
    from paper_2601_10729_b200.calibrate import b200_profile
    from paper_2601_10729_b200.core import RequestState
    from paper_2601_10729_b200.engine import RunConfig, Simulation
    from paper_2601_10729_b200.executor import B200Executor, ModelShape
    from paper_2601_10729_b200.metrics import collect_metrics
    from paper_2601_10729_b200.policies import PolicyKind, make_policy, plan_flexgen_plus
    from paper_2601_10729_b200.tp import HeadShard, TensorParallelExecutor, TensorParallelLlama

    cfg = CONFIGS["cfg4"]
    rank, world, local = _env_rank()
    local = local % max(1, torch.cuda.device_count())
    dist = None
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist  # noqa: F811

        dist.init_process_group(os.environ.get("OFB_DIST_BACKEND", "nccl"))
    dev = torch.device("cuda", local)
    tp = world if world > 1 else max(1, args.tp_emulate)
    shard = HeadShard(rank if world > 1 else 0, tp, cfg["hq"], cfg["hkv"])
    shape = ModelShape(cfg["layers"], shard.local_q, shard.local_kv)
    L, B, P = cfg["layers"], cfg["batch"], cfg["prompt"]
    outs = [args.cfg4_output + 2 * (i % 4) for i in range(B)]
    trace = workload.Trace(tuple(workload.TraceRequest(0, P, o) for o in outs),
                           {"config": "cfg4-serve"})
    cap = -(-(P + max(outs) + 1) // 16)
    slots = args.staging_slots
    wbytes = decoder_weight_bytes(cfg, shard)
    free_b, _ = torch.cuda.mem_get_info(dev)
    kv_budget = free_b - wbytes - B * slots * cap * shape.block_bytes - (8 << 30)
    if dist is not None:
        t = torch.tensor([kv_budget], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        kv_budget = int(t.item())
    budget = int(kv_budget // shape.block_bytes)
    h2d_peak, d2h_peak = _probe_link(dev)
    peaks = _measured_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6450.0)
    # B200 cost model: the weight stream of a layer joins its fixed cost
    layer_fixed = 0.012 + wbytes / L / (hbm_peak * 1e6)
    profile = b200_profile(L, shard.local_kv, budget, h2d_gbs=h2d_peak, layer_fixed_ms=layer_fixed)
    slo = defaults.default_slo(profile, scale=args.slo_scale)
    run_cfg = RunConfig(max_batch=B, batch_token_cap=B * (P + max(outs)))
    kind = PolicyKind(args.cfg4_policy)

    def policy():
        return make_policy(kind, profile, slo, max_batch=run_cfg.max_batch,
                           token_cap=run_cfg.batch_token_cap)

    head = {"metric": METRIC, "config": "cfg4-serve", "n_gpus": world, "tp": tp,
            "workload": (f"Llama-3.1-70B shape, {B} requests x {P}-token prompts arriving at t=0, "
                         f"outputs {min(outs)}-{max(outs)}, whole decoder step, policy {kind.value}"
                         + ("" if world > 1 else f"; rank 0's shard of TP{tp} on one GPU")),
            "policy": kind.value, "budget_blocks_per_rank": budget,
            "block_bytes_per_rank": shape.block_bytes, "weight_bytes_per_rank": wbytes,
            "slo": {"tpot_ms": slo.tpot_target_ms, "tbt_ms": slo.tbt_target_ms,
                    "scale": args.slo_scale, "source": "defaults.default_slo(profile)"},
            "profile": {"compute_base_ms": profile.compute_base_ms,
                        "compute_per_token_ms": profile.compute_per_token_ms,
                        "bandwidth_blocks_per_ms": profile.bandwidth_blocks_per_ms},
            "h2d_peak_gbs": h2d_peak, "d2h_peak_gbs": d2h_peak, "hbm_peak_gbs": hbm_peak}
    full_batch = [RequestState(id=i, arrival_time_ms=0.0, prompt_tokens=P,
                               target_output_tokens=o) for i, o in enumerate(outs)]
    first_plan = plan_flexgen_plus(full_batch, profile)
    n_off = sum(row.count(0) for row in first_plan.rows)
    host_need = n_off * cap * shape.block_bytes
    avail = _mem_available() // max(1, world)
    if host_need > 0.85 * avail:
        if rank == 0:
            print(json.dumps(dict(head, unavailable=(
                f"needs {host_need / 2**30:.0f} GiB of pinned host KV per rank "
                f"({n_off} offloaded slabs of {L * B}), {avail / 2**30:.0f} GiB available"))),
                flush=True)
        return
    t0 = time.perf_counter()
    model_log = Simulation(trace, policy(), profile, slo, run_cfg).execute()
    model_s = time.perf_counter() - t0
    ex = B200Executor(shape, device=dev, device_blocks=budget + B * slots * cap + 64,
                      host_blocks=int(n_off * cap * 1.25) + 64, staging_slots=slots,
                      copy_streams=args.copy_streams, seed=rank)
    dec = TensorParallelLlama(ex, shard, cfg["hidden"], cfg["intermediate"], c1=args.c1,
                              max_batch=B)
    tex = TensorParallelExecutor(dec, seed=0)
    out = dict(head, offloaded_slabs_first_plan=n_off,
               host_control_ms_per_step_model=model_s * 1e3 / max(1, sum(
                   r["kind"] == "step" for r in model_log)))
    # warm-up: a two-request trace through the same executor (cuBLAS heuristics,
    # module loading, first-launch costs stay out of the measured runs)
    warm = workload.Trace((workload.TraceRequest(0, 1000, 3), workload.TraceRequest(0, 900, 4)), {})
    Simulation(warm, policy(), profile, slo, run_cfg, executor=tex).execute()
    modes = [m.strip() for m in args.cfg4_modes.split(",") if m.strip()]
    for mode in modes:
        tex.steps = 0
        with ClockSampler(local) as clocks:
            t0 = time.perf_counter()
            log = Simulation(trace, policy(), profile, slo, run_cfg, executor=tex,
                             mode=mode).execute()
            wall_s = time.perf_counter() - t0
        steps = [r for r in log if r["kind"] == "step"]
        gpu_ms = [r["payload"]["measured_us"] / 1e3 for r in steps]
        tokens = sum(len(r["payload"]["ids"]) for r in steps)
        rep = collect_metrics(log)
        first = steps[0]["payload"]
        rows, ids = first["rows"], first["ids"]
        T = {r: P for r in ids}
        host_alg = sum(row.count(0) * -(-T[i] // 16) for i, row in zip(ids, rows)) * shape.block_bytes
        hbm_alg = (sum(row.count(1) * T[i] for i, row in zip(ids, rows)) * shape.kv_bytes_per_token
                   + wbytes)
        roof_ms = max(hbm_alg / (hbm_peak * 1e9), host_alg / (h2d_peak * 1e9)) * 1e3
        # steady state at the full batch: the first step also pays one-time costs
        # (first-touch of staging / workspaces), so it is reported separately
        full = [g for r, g in zip(steps, gpu_ms) if len(r["payload"]["ids"]) == B][1:]
        full_ms = statistics.median(full) if full else gpu_ms[0]
        span_us = steps[-1]["time_us"] + steps[-1]["payload"].get(
            "wall_us", steps[-1]["payload"]["measured_us"]) - steps[0]["time_us"]
        hist = {}
        for r in steps:
            hist[len(r["payload"]["ids"])] = hist.get(len(r["payload"]["ids"]), 0) + 1
        rec = {"steps": len(steps), "tokens": tokens, "gpu_ms_total": sum(gpu_ms),
               "tokens_per_s_device": tokens / (sum(gpu_ms) * 1e-3),
               "tokens_per_s_clock": (tokens / (span_us * 1e-6) if span_us > 0 and mode != "parity"
                                      else None),
               "wall_s": wall_s, "step_ms_median": statistics.median(gpu_ms),
               "tpot_attainment": rep.tpot_attainment, "tbt_attainment": rep.tbt_attainment,
               "tpot_p95_ms": rep.tpot_p95_ms, "tbt_p95_ms": rep.tbt_p95_ms,
               "batch_histogram": hist, "replans": rep.replans, "pauses": rep.pauses,
               "preemptions": rep.preemptions, "migrated": dict(ex.migrated),
               "step_roofline": {"offloaded_slabs": sum(row.count(0) for row in rows),
                                 "bound": "host_link" if host_alg / h2d_peak > hbm_alg / hbm_peak
                                 else "hbm",
                                 "host_alg_bytes": host_alg, "hbm_alg_bytes": hbm_alg,
                                 "roofline_ms": roof_ms,
                                 "measured_ms_full_batch_median": full_ms,
                                 "full_batch_steps": len(full),
                                 "achieved_frac": roof_ms / full_ms,
                                 # per-GPU rates over the full-batch median step
                                 "hbm_gbs_per_gpu": hbm_alg / (full_ms * 1e-3) / 1e9,
                                 "host_link_gbs_per_gpu": host_alg / (full_ms * 1e-3) / 1e9,
                                 "first_step_ms": gpu_ms[0]},
               "clocks": clocks.summary()}
        if "wall_us" in steps[0]["payload"]:
            walls = [r["payload"]["wall_us"] / 1e3 for r in steps]
            rec["host_ms_per_step_median"] = statistics.median(
                w - g for w, g in zip(walls, gpu_ms))
        if mode == "parity":
            stripped = [dict(r, payload={k: v for k, v in r["payload"].items()
                                         if k not in ("measured_us", "wall_us")})
                        if r["kind"] == "step" else r for r in log]
            rec["decisions_match_model_run"] = stripped == model_log
            rec["model_tpot_attainment"] = collect_metrics(model_log).tpot_attainment
        out[mode] = rec
        if rank == 0:
            print(json.dumps({"mode": mode, **rec}), file=sys.stderr, flush=True)
    tex.close()
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS) + ["cfg3", "cfg3-policies", "cfg4-serve",
                                                           "cfg5"],
                    default="cfg2")
    ap.add_argument("--slo-scale", type=float, default=1.5)
    ap.add_argument("--cfg3-requests", type=int, default=24)
    ap.add_argument("--cfg3-rate", type=float, default=30.0,
                    help="cfg3 arrival rate (requests/s; SURVEY.md 8(d): 30)")
    ap.add_argument("--cfg3-output-median", type=int, default=256)
    ap.add_argument("--cfg3-budget-blocks", type=int, default=655360,
                    help="cfg3 HBM pool in 64 KiB blocks (SURVEY.md 8(d): a 40 GiB pool)")
    ap.add_argument("--cfg3-calibrate", action="store_true",
                    help="cfg3: SystemProfile measured on this GPU (K1 slope/intercept, link)")
    ap.add_argument("--cfg3-policies", default="",
                    help="comma list for --config cfg3-policies (default: every policy)")
    ap.add_argument("--staging-slots", type=int, default=2,
                    help="1 = reference single-slot launch rule, 2 = double-buffered staging")
    ap.add_argument("--copy-streams", type=int, default=16)
    ap.add_argument("--layer-events", choices=["separate", "inline"], default="inline",
                    help="per-layer K1 / per-copy CUDA events inside the timed steps (default; free "
                         "when the step is link-bound) or in a separate instrumented pass - an event "
                         "between two kernels breaks their programmatic-dependent-launch overlap, "
                         "which costs ~6%% on HBM-bound steps (cfg4, cfg2r)")
    ap.add_argument("--ref-seconds", type=float, default=3.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--decoder", choices=["attn", "full"], default=None,
                    help="full: whole decoder step (QKV / MLP weights streamed); default full for "
                         "cfg4, attention path for the others")
    ap.add_argument("--c1", choices=["k6", "nccl"], default="k6",
                    help="TP exchange: K6 (projection fused with the all-reduce over peer memory) "
                         "or cuBLAS projection + NCCL all-reduce")
    ap.add_argument("--tp-emulate", type=int, default=1,
                    help="run rank 0's KV-head shard of a TP-N deployment on one GPU")
    ap.add_argument("--sweep-max-tokens", type=int, default=1048576,
                    help="cfg5: largest B x T swept (KV bytes = tokens x 128 KiB)")
    ap.add_argument("--cfg4-output", type=int, default=16,
                    help="cfg4-serve: output tokens per request (+0/2/4/6 by request)")
    ap.add_argument("--cfg4-policy", default="flexgen_plus",
                    help="cfg4-serve: a tractable plan source at B=32, L=80 (SURVEY.md 8(d))")
    ap.add_argument("--cfg4-modes", default="parity,live-wall",
                    help="cfg4-serve: engine clock modes to run (engine.MODES)")
    args = ap.parse_args()
    if args.config == "cfg4-serve":
        return run_cfg4_serve(args)
    if args.config == "cfg5":
        return run_reconfig(args)
    if args.config == "cfg3":
        return run_cfg3(args)
    if args.config == "cfg3-policies":
        return run_cfg3_policies(args)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference_arm(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
