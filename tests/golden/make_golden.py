"""Generate golden parity fixtures by running the REFERENCE (kvsim) itself.

Run in the build container, where /root/reference exists:
    python tests/golden/make_golden.py
Outputs (committed, small): tests/golden/*.json.  Floats are stored as
``float.hex`` strings so bit-exactness can be asserted anywhere (the GPU box
has no /root/reference).  Nothing here is imported by the product package.
"""

from __future__ import annotations

import hashlib
import json
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

import kvsim  # noqa: E402  (the reference)
from kvsim import defaults, workload  # noqa: E402
from kvsim.core import PlacementMatrix, RequestState, SloConfig, SystemProfile  # noqa: E402
from kvsim.engine import BlockTable, RunConfig, Simulation, apply_plan  # noqa: E402
from kvsim.latency import _simulate_stalls, batch_decode_latency_fast  # noqa: E402
from kvsim.planner import (Infeasible, forecast_violations, solve,  # noqa: E402
                           solve_capacity_only, solve_one_step_ahead)
from kvsim.policies import PolicyKind, PolicyOptions, make_policy  # noqa: E402


def hx(x: float) -> str:
    return float(x).hex()


def req(rid, prompt, generated=0, output=400, arrival=0.0, deposit=0):
    r = RequestState(id=rid, arrival_time_ms=arrival, prompt_tokens=prompt,
                     target_output_tokens=output)
    r.generated_tokens = generated
    r.deposit_balance = deposit
    r.sync_blocks()
    return r


def req_json(r):
    return {"id": r.id, "prompt": r.prompt_tokens, "generated": r.generated_tokens,
            "output": r.target_output_tokens, "arrival": r.arrival_time_ms,
            "deposit": r.deposit_balance}


def profile_json(p: SystemProfile):
    return {"num_layers": p.num_layers, "compute_base_ms": hx(p.compute_base_ms),
            "compute_per_token_ms": hx(p.compute_per_token_ms),
            "bandwidth_blocks_per_ms": hx(p.bandwidth_blocks_per_ms),
            "gpu_block_budget": p.gpu_block_budget, "block_size": p.block_size,
            "prefill_per_token_ms": hx(p.prefill_per_token_ms), "ewma_decay": hx(p.ewma_decay)}


def slo_json(s: SloConfig):
    return {"tbt": hx(s.tbt_target_ms), "tpot": hx(s.tpot_target_ms),
            "cap": hx(s.violation_cap), "wmin": s.window_min, "wmax": s.window_max,
            "theta": hx(s.profile_mismatch_threshold)}


def plan_json(plan):
    if isinstance(plan, Infeasible):
        return {"infeasible": plan.reason}
    lat = plan.predicted_latency
    return {"rows": [list(r) for r in plan.placement.rows], "window": plan.decode_window,
            "expiry": plan.expiry_step, "latency": hx(lat.total_latency_ms),
            "stalls": [hx(s) for s in lat.per_layer_stall_ms], "fetched": lat.blocks_fetched}


def schedule_vectors(rng):
    cases = []
    for _ in range(400):
        L = rng.randint(1, 40)
        n = rng.randint(1, 6)
        sizes = [rng.randint(1, 300) for _ in range(n)]
        offl = [[rng.random() < rng.choice((0.2, 0.5, 0.8)) for _ in range(L)] for _ in range(n)]
        comp = rng.choice([0.01, 0.25, 0.5, 1.0, 1.5, 3.0, rng.uniform(0.001, 5.0)])
        bw = rng.choice([1.0, 3.0, 7.0, 220.0, rng.uniform(0.5, 500.0)])
        lists = [[l + 1 for l in range(L) if o[l]] for o in offl]
        stalls = _simulate_stalls(sizes, lists, L, comp, bw, exact=False)
        total = comp * L + sum(stalls)
        cases.append({"L": L, "sizes": sizes, "offloaded": [[int(v) for v in o] for o in offl],
                      "comp": hx(comp), "bw": hx(bw), "stalls": [hx(s) for s in stalls],
                      "total": hx(total)})
    return cases


def solve_vectors(rng):
    out = []
    layer_choices = [4, 6, 9, 10, 12, 32]
    for i in range(120):
        L = rng.choice(layer_choices)
        B = rng.randint(1, 3 if L >= 12 else 4)
        batch = [req(r, rng.randint(10, 700), generated=rng.randint(0, 30),
                     arrival=float(rng.randint(0, 5)), deposit=rng.randint(0, 3)) for r in range(B)]
        total_kv = sum(r.blocks_per_layer for r in batch) * L
        budget = max(max(r.blocks_per_layer for r in batch) + 2, int(total_kv * rng.uniform(0.3, 1.2)))
        prof = SystemProfile(L, rng.choice([0.2, 0.5, 1.0]), rng.choice([0.0, 0.0002, 0.001]),
                             rng.choice([2.0, 3.0, 10.0, 50.0]), budget, 16)
        lat_all = batch_decode_latency_fast(PlacementMatrix.all_resident([r.id for r in batch], L),
                                            batch, prof).total_latency_ms
        slo = SloConfig(tbt_target_ms=lat_all * rng.choice([1.0, 1.5, 3.0, 10.0]),
                        tpot_target_ms=lat_all * 2, violation_cap=rng.choice([0.5, 1.0, 2.0]),
                        window_min=rng.randint(1, 4), window_max=rng.randint(4, 16))
        paused = tuple(req(100 + j, rng.randint(10, 300), deposit=rng.randint(0, 2))
                       for j in range(rng.choice([0, 0, 1])))
        snap = None
        if rng.random() < 0.5:
            snap = {r.id: rng.uniform(0, 3) for r in batch + list(paused)}
        step = rng.randint(1, 50)
        res = solve(batch, prof, slo, step, paused=paused, deposit_snapshot=snap)
        ahead = solve_one_step_ahead(batch, prof, slo, step, paused=paused, deposit_snapshot=snap)
        cap = solve_capacity_only(batch, prof, slo, step)
        fc = None
        if not isinstance(res, Infeasible):
            f = forecast_violations(res.placement, batch, prof, slo, slo.window_max,
                                    deposit_snapshot=snap, paused=paused)
            fc = {"fails": list(f.per_step_failures), "truncated": f.truncated_at}
        out.append({"profile": profile_json(prof), "slo": slo_json(slo),
                    "batch": [req_json(r) for r in batch], "paused": [req_json(p) for p in paused],
                    "snapshot": None if snap is None else {str(k): hx(v) for k, v in snap.items()},
                    "step": step, "solve": plan_json(res), "ahead": plan_json(ahead),
                    "capacity_only": plan_json(cap), "forecast": fc})
    return out


def table_vectors(rng):
    """apply_plan / pause / evict sequences -> block-table snapshots."""
    out = []
    for _ in range(40):
        L = rng.randint(2, 8)
        prof = SystemProfile(L, 1.0, 0.0, rng.choice([2.0, 5.0]), rng.randint(40, 200), 16)
        table = BlockTable(L, prof.gpu_block_budget)
        ids = list(range(rng.randint(1, 4)))
        pool = {i: req(i, rng.randint(10, 120)) for i in ids}
        initial = {str(i): req_json(r) for i, r in pool.items()}
        ops = []
        batch = list(pool.values())
        for _step in range(rng.randint(3, 10)):
            action = rng.random()
            if action < 0.2 and len(batch) > 1:
                victim = batch.pop(rng.randrange(len(batch)))
                table.mark_removable(victim.id, victim.blocks_per_layer)
                ops.append({"op": "pause", "id": victim.id})
                continue
            if action < 0.3:
                paused = [i for i in pool if pool[i] not in batch]
                if paused:
                    back = pool[paused[0]]
                    batch.append(back)
                    table.clear_pause(back.id)
                    ops.append({"op": "resume", "id": back.id})
                    continue
            rows = tuple(tuple(rng.choice((0, 1, 1)) for _ in range(L)) for _ in batch)
            pm = PlacementMatrix(tuple(r.id for r in batch), L, rows)
            from kvsim.core import Plan
            plan = Plan(pm, batch_decode_latency_fast(pm, batch, prof), 1, None)
            try:
                charge = apply_plan(plan, table, batch, prof)
                ops.append({"op": "apply", "ids": [r.id for r in batch], "rows": [list(r) for r in rows],
                            "charge": hx(charge),
                            "locations": {str(k): "".join(v) for k, v in table.locations.items()},
                            "blocks": {str(k): v for k, v in table.blocks.items()},
                            "buffer": table.buffer_reservation})
            except Exception as exc:  # CapacityError
                ops.append({"op": "apply", "ids": [r.id for r in batch], "rows": [list(r) for r in rows],
                            "error": type(exc).__name__})
                break
            for r in batch:
                r.record_generated_token()
                table.blocks[r.id] = r.blocks_per_layer
        out.append({"profile": profile_json(prof),
                    "requests": initial, "ops": ops})
    return out


def log_digest(log):
    blob = json.dumps(log, sort_keys=True).encode()
    return hashlib.sha256(blob).hexdigest()


def simulation_vectors():
    """Whole-engine runs: sha256 of the full event log + headline counts."""
    out = []
    cells = []
    trace_small = workload.generate(3, 400.0, 1.0, workload.LengthSpec(
        prompt_median=120, output_median=12, max_prompt=600, max_output=40), 12)
    for pk in PolicyKind:
        cells.append(("small", trace_small, defaults.DEFAULT_PROFILE, 1.5, pk, RunConfig()))
    suite = defaults.make_suite_trace(11, count=40)
    for pk in (PolicyKind.ORBIT, PolicyKind.FLEXGEN_PLUS, PolicyKind.DYNAMIC_HEURISTIC):
        cells.append(("suite11", suite, defaults.DEFAULT_PROFILE, 1.0, pk, RunConfig()))
    stress = defaults.make_stress_trace(12, count=25)
    cells.append(("stress12", stress, defaults.DEFAULT_PROFILE, 1.5, PolicyKind.ORBIT,
                  RunConfig(scheduler="srtf", solver_overhead_ms=5.0)))
    cells.append(("stress12-shortest", stress, defaults.DEFAULT_PROFILE, 1.0, PolicyKind.ORBIT,
                  RunConfig(seed=7)))
    for name, trace, prof, scale, pk, cfg in cells:
        slo = defaults.default_slo(prof, scale=scale)
        opts = defaults.suite_policy_options(pk, victim="shortest" if "shortest" in name else "largest")
        policy = make_policy(pk, prof, slo, opts, max_batch=cfg.max_batch, token_cap=cfg.batch_token_cap)
        log = Simulation(trace, policy, prof, slo, cfg).execute()
        rep = kvsim.collect_metrics(log)
        entry = {"cell": name, "policy": pk.value, "scale": scale, "config": cfg.__dict__,
                 "trace": {"text": workload.serialize(trace)}, "profile": profile_json(prof),
                 "victim": opts.victim, "worst_case_tokens": opts.worst_case_tokens,
                 "digest": log_digest(log), "records": len(log),
                 "report": json.loads(rep.to_json())}
        if name == "small" and pk == PolicyKind.ORBIT:
            entry["steps"] = [r for r in log if r["kind"] in ("step", "pause", "resume", "replan")]
        out.append(entry)
    return out


def toy_cfg1():
    """BASELINE config 1: the reference plan the GPU path executes."""
    prof = SystemProfile(num_layers=4, compute_base_ms=0.01,
                         compute_per_token_ms=1024 / 6.5e12 * 1e3,
                         bandwidth_blocks_per_ms=55e9 / 16384 / 1e3, gpu_block_budget=2560,
                         block_size=16)
    slo = SloConfig(50.0, 50.0, window_min=4, window_max=32)
    batch = [req(i, 4088, output=64) for i in range(4)]
    plan = solve(batch, prof, slo, 1)
    return {"profile": profile_json(prof), "slo": slo_json(slo),
            "batch": [req_json(r) for r in batch], "plan": plan_json(plan)}


def main():
    rng = random.Random(20260117)
    fixtures = {
        "schedule_vectors.json": schedule_vectors(rng),
        "solve_vectors.json": solve_vectors(rng),
        "table_vectors.json": table_vectors(rng),
        "simulation_vectors.json": simulation_vectors(),
        "cfg1_plan.json": toy_cfg1(),
    }
    for name, data in fixtures.items():
        (OUT / name).write_text(json.dumps(data, sort_keys=True, separators=(",", ":")) + "\n")
        print(name, (OUT / name).stat().st_size, "bytes")


if __name__ == "__main__":
    main()
