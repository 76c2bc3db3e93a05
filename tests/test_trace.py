"""The trace contract (schedule.py:334-402): validate_trace on synthetic traces (CPU) and on the
device-timed traces that run() returns (GPU), for every order, with the ledger at 2 workers."""
import numpy as np
import pytest

from paper_2511_16174_b200 import (CommLedger, PipelineConfig, TraceEvent, mean_idle_fraction,
                                   validate_trace)


def ev(w, stage, t0, t1):
    return TraceEvent(worker=w, stage=stage, block=0, t_start=t0, t_end=t1)


def test_valid_trace_and_idle():
    events = [ev(0, "SBR", 0, 10), ev(1, "SBR", 10, 20), ev(0, "BC", 20, 25),
              ev(1, "BC", 25, 30), ev(-1, "Solver", 30, 40), ev(0, "BC-Back", 30, 45),
              ev(0, "FinalMultiply", 45, 50), ev(1, "FinalMultiply", 40, 50)]
    led = CommLedger()
    led.record(0, 1, "BC", 8)
    validate_trace(events, 2, led)
    assert 0.0 <= mean_idle_fraction(events, 2) < 1.0


@pytest.mark.parametrize("events,msg", [
    ([ev(0, "SBR", 0, 10), ev(0, "BC", 5, 12)], "overlaps"),
    ([ev(0, "SBR", 0, 10), ev(1, "SBR", 5, 20)], "chain broken"),
    ([ev(0, "BC", 0, 10), ev(1, "BC-Back", 5, 20)], "before the reflector gather"),
    ([ev(-1, "Solver", 0, 10), ev(0, "FinalMultiply", 5, 20)], "before the solver"),
])
def test_violations(events, msg):
    with pytest.raises(ValueError, match=msg):
        validate_trace(events, 2)


def test_ledger_boundary_messages():
    led = CommLedger()
    led.record(0, 1, "BC", 8)
    led.record(0, 1, "BC", 8)
    with pytest.raises(ValueError, match="exactly one overlap message"):
        validate_trace([], 2, led)


@pytest.mark.gpu
@pytest.mark.parametrize("order", ["pipelined", "sequential", "conventional"])
@pytest.mark.parametrize("workers", [1, 2])
def test_run_trace_is_valid(order, workers):
    import paper_2511_16174_b200 as pkg
    g = np.random.default_rng(3).standard_normal((300, 300))
    a = (g + g.T) / 2
    res, events, ledger, counter = pkg.run(a, PipelineConfig(workers=workers, b=32, order=order))
    validate_trace(events, workers, ledger)
    assert {e.stage for e in events} >= {"SBR", "BC", "Solver", "SBR-Back", "BC-Back"}
