"""The Fig.-3 fixture's additional golden values SURVEY.md section 4 records from the
reference (measured there, not asserted by the reference's own tests), pinned here
for this package - both solve paths (native C++ and numpy restatement).

Fixture (reference tests/conftest.py): 9 layers, 1 ms per layer, 3 blocks/ms,
70-block budget, prompts 34 / 81 (3 / 6 blocks), window 1.
"""

import pytest

from paper_2601_10729_b200 import planner
from paper_2601_10729_b200.core import PlacementMatrix, RequestState, SloConfig, SystemProfile
from paper_2601_10729_b200.latency import batch_decode_latency


def _req(rid, prompt, generated):
    r = RequestState(id=rid, arrival_time_ms=0.0, prompt_tokens=prompt, target_output_tokens=400,
                     block_size=16)
    r.generated_tokens = generated
    r.sync_blocks()
    return r


PROFILE = SystemProfile(num_layers=9, compute_base_ms=1.0, compute_per_token_ms=0.0,
                        bandwidth_blocks_per_ms=3.0, gpu_block_budget=70, block_size=16)
SLO = SloConfig(tbt_target_ms=1e6, tpot_target_ms=1e6, window_min=1, window_max=1)
ROWS_B = ((1, 1, 1, 1, 1, 1, 1, 1, 1), (1, 1, 0, 1, 1, 0, 1, 1, 0))
ROWS_C = ((1, 1, 1, 0, 1, 1, 1, 0, 1), (1, 1, 0, 1, 1, 0, 1, 1, 0))


@pytest.fixture(params=["native", "python"])
def solver(request):
    prev = planner.SOLVER
    planner.SOLVER = request.param
    yield request.param
    planner.SOLVER = prev


def test_solve_step1_is_placement_b(solver):
    batch = [_req(0, 34, 0), _req(1, 81, 0)]
    plan = planner.solve(batch, PROFILE, SLO, current_step=1)
    assert plan.placement.rows == ROWS_B
    assert plan.predicted_latency.total_stall_ms == 0.0
    assert plan.predicted_latency.total_latency_ms == 9.0


def test_solve_step16_is_placement_c(solver):
    batch = [_req(0, 34, 15), _req(1, 81, 15)]
    plan = planner.solve(batch, PROFILE, SLO, current_step=16)
    assert plan.placement.rows == ROWS_C
    # reference: total_latency_ms 11.333333333333332, stall units 6.999999999999999
    assert plan.predicted_latency.total_latency_ms.hex() == "0x1.6aaaaaaaaaaaap+3"
    assert plan.predicted_latency.stall_transfer_units == 6.999999999999999
    assert plan.decode_window == 1 and plan.expiry_step == 17


def test_placement_c_stalls_6_then_7_units():
    """The divergence SPEC.md:616 anticipated: the paper says 0 and 2 stalls.
    Values (float hex) as the reference's batch_decode_latency returns them."""
    pc = PlacementMatrix((0, 1), 9, ROWS_C)
    for generated, units, total_hex in ((0, 6.0, "0x1.6000000000000p+3"),
                                        (15, 7.0, "0x1.6aaaaaaaaaaabp+3")):
        lat = batch_decode_latency(pc, [_req(0, 34, generated), _req(1, 81, generated)], PROFILE)
        assert lat.stall_transfer_units == units
        assert lat.total_latency_ms.hex() == total_hex
