"""The cost model and schedule simulator (reference schedule.py:82-332, tests/test_schedule.py
:73-215) and the B200-refit model."""
import numpy as np
import pytest

from paper_2511_16174_b200 import PipelineConfig
from paper_2511_16174_b200.costmodel import (CostModel, b200_model, calibrated_model, load_model,
                                             simulate, unit_model)
from paper_2511_16174_b200.messaging import CommLedger
from paper_2511_16174_b200.schedule import validate_trace


def test_cost_model_durations():
    m = CostModel(p=100.0, q=10.0, stage_rate={"BC": 0.5})
    assert m.duration("SBR", 200) == 2.0
    assert m.duration("BC", 200) == 4.0
    assert m.duration("SBR", 200, words=50) == 7.0
    assert m.comm_seconds(30) == 3.0
    u = unit_model()
    assert u.duration("SBR", 10 ** 12, words=10 ** 9) == 1.0 and u.comm_seconds(10 ** 9) == 0.0


def test_unit_simulation_hand_checked():
    # one tick per task: the pipelined order overlaps the chase with basis generation
    _, sp = simulate(unit_model(), PipelineConfig(workers=2, b=32, order="pipelined"), 512)
    _, ss = simulate(unit_model(), PipelineConfig(workers=2, b=32, order="sequential"), 512)
    assert (sp, ss) == (6.0, 7.0)
    _, sp = simulate(unit_model(), PipelineConfig(workers=1, b=32, order="pipelined"), 256)
    _, ss = simulate(unit_model(), PipelineConfig(workers=1, b=32, order="sequential"), 256)
    assert sp == ss == 5.0


@pytest.mark.parametrize("model", [calibrated_model(), b200_model()])
def test_simulated_traces_validate_and_pipelining_helps(model):
    for seed in range(15):
        rng = np.random.default_rng(seed)
        w = int(rng.integers(1, 7))
        b = int(rng.integers(2, 33))
        n = int(rng.integers(max(8 * w, 4 * b), 1500))
        skew = float(rng.uniform(0.0, 0.05))
        spans = {}
        for order in ("pipelined", "sequential"):
            ledger = CommLedger()
            events, spans[order] = simulate(model, PipelineConfig(workers=w, b=b, order=order,
                                                                  back_skew=skew), n, ledger)
            validate_trace(events, w, ledger)
        assert spans["pipelined"] <= spans["sequential"]


def test_simulate_rejects_conventional_and_is_deterministic():
    with pytest.raises(ValueError, match="pipelined or sequential"):
        simulate(unit_model(), PipelineConfig(workers=2, b=8, order="conventional"), 64)
    cfg = PipelineConfig(workers=3, b=16, order="pipelined", back_skew=0.03)
    assert simulate(calibrated_model(), cfg, 777) == simulate(calibrated_model(), cfg, 777)


def test_calibrated_ratio_improves_with_workers():
    prev = 1.0
    for w in (1, 2, 4):
        _, sp = simulate(calibrated_model(), PipelineConfig(workers=w, b=32, order="pipelined"), 2048)
        _, ss = simulate(calibrated_model(), PipelineConfig(workers=w, b=32, order="sequential"), 2048)
        assert sp / ss <= prev + 1e-12
        prev = sp / ss
    assert prev < 0.9


def test_b200_model_reproduces_measured_single_gpu_stages():
    """The refit rates give back the measured stage seconds at the fit point, and the model
    prices one worker at the headline size near the measured sequential wall."""
    from paper_2511_16174_b200.costmodel import (B200_STAGE_SECONDS, bc_back_macs,
                                                 sbr_macs_for_range)
    m = b200_model()
    n, b = B200_STAGE_SECONDS["n"], B200_STAGE_SECONDS["b"]
    assert abs(m.duration("SBR", sbr_macs_for_range(n, b, (0, n))) - B200_STAGE_SECONDS["SBR"]) < 1e-9
    assert abs(m.duration("BC-Back", bc_back_macs(n, n)) - B200_STAGE_SECONDS["BC-Back"]) < 1e-9
    _, span = simulate(m, PipelineConfig(workers=1, b=b, order="sequential"), n)
    S = B200_STAGE_SECONDS
    want = S["SBR"] + S["BC"] + max(S["SBR-Back"], S["Solver"]) + S["BC-Back"] + S["FinalMultiply"]
    assert abs(span - want) < 0.1  # + the words / q terms (SBR broadcasts, Q rows), ~0.06 s
    assert load_model("b200").stage_rate == m.stage_rate
