"""Stage cost model and schedule simulator (reference schedule.py:82-332), with a B200 model.

The reference prices each stage as multiply-adds / (p * rate[stage]) + words / q and plays the
pipelined or sequential stage graph forward (`simulate`).  The MAC formulas are the reference's
own (its FlopCounter conventions: SBR rounds, 7 b^2 per chase step, m n^2 for BC-Back and the
final multiply, 3.6 n^3 for the implicit-QR solver), so a model is just (p, q, rates).

`b200_model()` refits the rates to this build on one B200: p is the FP64 DMMA peak in MAC/s,
q the measured NVLink peer bandwidth in words/s, and each stage's rate is the reference-formula
MACs of that stage divided by (p x its measured B200 seconds) at n = 49152 -- so the simulator
answers "what would the reference's pipeline look like at B200 stage speeds", and a rate above
1 just means the stage needs fewer operations on the device than the reference's count (e.g. the
divide and conquer against the 3.6 n^3 QR count).
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field

from .messaging import HOST, TraceEvent
from .schedule import back_plan_sizes, partition

SIM_SCALE = 1_000_000  # integer trace ticks per model time unit (schedule.py SIM_SCALE)
STAGES = ("SBR", "BC", "SBR-Back", "BC-Back", "Solver", "FinalMultiply")


# ------------------------------------------------------------------ the reference's MAC counts
def _rounds(n: int, b: int):
    c0 = 0
    while c0 < n - b:
        yield c0, min(b, n - b - c0)
        c0 += b


def sbr_macs_for_range(n: int, b: int, cols) -> int:
    """Panel rounds owned by a column range: 2 m^2 pw + 4 m pw^2 each (schedule.py:84-99)."""
    lo, hi = cols
    return sum(2 * (n - c0 - b) ** 2 * pw + 4 * (n - c0 - b) * pw * pw
               for c0, pw in _rounds(n, b) if lo <= c0 < hi)


def sbr_words_for_range(n: int, b: int, cols) -> int:
    """Broadcast words of the rounds a range owns, 3 m pw each (schedule.py:102-113)."""
    lo, hi = cols
    return sum(3 * (n - c0 - b) * pw for c0, pw in _rounds(n, b) if lo <= c0 < hi)


def bc_macs_for_range(n: int, b: int, cols) -> int:
    """7 b^2 per chase step of the range's sweeps (schedule.py:116-122)."""
    lo, hi = cols
    return sum(7 * b * b * ((n - 3 - i) // b + 1) for i in range(lo, min(hi, n - 2)))


def sbr_back_macs(n: int, b: int, m: int) -> int:
    return sum(2 * m * (n - c0 - b) * pw for c0, pw in _rounds(n, b))


def bc_back_macs(n: int, m: int) -> int:
    return m * n * n


def solver_macs(n: int) -> int:
    return int(3.6 * n ** 3)


def final_macs(n: int, m: int) -> int:
    return m * n * n


# ------------------------------------------------------------------ models
@dataclass
class CostModel:
    """duration = macs / (p * stage_rate[stage]) + words / q; unit=True: one tick per task and
    free communication (the hand-checkable model)."""

    p: float = 1.0e10
    q: float = 1.25e9
    stage_rate: dict = field(default_factory=dict)
    unit: bool = False

    def duration(self, stage: str, macs: int, words: int = 0) -> float:
        if self.unit:
            return 1.0
        return macs / (self.p * self.stage_rate.get(stage, 1.0)) + words / self.q

    def comm_seconds(self, words: int) -> float:
        return 0.0 if self.unit else words / self.q


def unit_model() -> CostModel:
    return CostModel(unit=True)


def calibrated_model() -> CostModel:
    """The reference's CPU-shaped defaults (schedule.py:180-202)."""
    return CostModel(p=2.0e10, q=1.0e10,
                     stage_rate={"SBR": 1.0, "BC": 0.05, "SBR-Back": 1.0, "BC-Back": 0.15,
                                 "Solver": 10.0, "FinalMultiply": 1.0})


# measured on one B200 at n = 49152, b = 32 (bench.py stage times, profiles/r02_*; the
# pipelined-order stages SBR-Back / FinalMultiply at their own measured rates)
B200_STAGE_SECONDS = {"n": 49152, "b": 32, "SBR": 6.15, "BC": 1.10, "SBR-Back": 5.3,
                      "BC-Back": 9.0, "Solver": 3.9, "FinalMultiply": 7.0}
B200_DMMA_MACS = 37.17e12 / 2     # FP64 DMMA peak, MAC/s (profiles/r01_fp64_peaks.json)
B200_PEER_WORDS = 770e9 / 8       # measured NVLink peer copy, words/s (B200_PROFILING.md)


def b200_model(seconds: dict | None = None) -> CostModel:
    """Rates refit from measured B200 stage times: rate = formula MACs / (p * seconds)."""
    s = dict(B200_STAGE_SECONDS if seconds is None else seconds)
    n, b = int(s["n"]), int(s["b"])
    whole = (0, n)
    macs = {"SBR": sbr_macs_for_range(n, b, whole), "BC": bc_macs_for_range(n, b, whole),
            "SBR-Back": sbr_back_macs(n, b, n), "BC-Back": bc_back_macs(n, n),
            "Solver": solver_macs(n), "FinalMultiply": final_macs(n, n)}
    p = B200_DMMA_MACS
    return CostModel(p=p, q=B200_PEER_WORDS,
                     stage_rate={k: macs[k] / (p * s[k]) for k in STAGES})


def load_model(spec: str) -> CostModel:
    """'calibrated', 'unit', 'b200', or a JSON file {p, q, stage_rate} (cli.py model option)."""
    if spec == "calibrated":
        return calibrated_model()
    if spec == "unit":
        return unit_model()
    if spec == "b200":
        return b200_model()
    try:
        with open(spec) as fh:
            d = json.load(fh)
        return CostModel(p=float(d["p"]), q=float(d["q"]),
                         stage_rate={k: float(v) for k, v in d.get("stage_rate", {}).items()})
    except (OSError, KeyError, TypeError, ValueError) as exc:
        raise ValueError(f"malformed cost model {spec!r}: {exc}") from exc


# ------------------------------------------------------------------ the stage graph
def simulate(model: CostModel, cfg, n: int, ledger=None):
    """Play the stage graph forward (schedule.py:205-332): returns (events, makespan).

    Rules (the runtime's): SBR owner phases chain worker to worker; the relayed chase starts on
    worker i once its SBR phase and worker i-1's chase are done (sequential order: after the
    whole SBR); the solver starts after the last chase; SBR-Back fills the gap between a
    worker's SBR phase and its chase, the rest after its chase (sequential: all after the last
    chase); BC-Back after the U gather (= the last chase) and the worker's SBR-Back; the final
    multiply after BC-Back and the solver.  Sequential order puts barriers between SBR-Back /
    solver, BC-Back and the final multiply.  Every start is a max of finish times, so the
    makespan is monotone in every cost and the schedule deterministic."""
    if cfg.order not in ("pipelined", "sequential"):
        raise ValueError(f"simulate supports pipelined or sequential, not {cfg.order!r}")
    W, b = cfg.workers, cfg.b
    seq = cfg.order == "sequential"
    cols = partition(n, W)
    rows = back_plan_sizes(n, W, cfg.back_skew)
    words_sbr = [sbr_words_for_range(n, b, c) for c in cols]
    words_bc = [(2 * b * b if i < W - 1 else 0) + (n - cols[i][1]) * (2 * b + 1)
                for i in range(W)]
    d_sbr = [model.duration("SBR", sbr_macs_for_range(n, b, cols[i]), words_sbr[i])
             for i in range(W)]
    d_bc = [model.duration("BC", bc_macs_for_range(n, b, cols[i]), words_bc[i]) for i in range(W)]
    d_gen = [model.duration("SBR-Back", sbr_back_macs(n, b, m)) for m in rows]
    d_bb = [model.duration("BC-Back", bc_back_macs(n, m)) for m in rows]
    d_fm = [model.duration("FinalMultiply", final_macs(n, m), m * n) for m in rows]
    d_solve = model.duration("Solver", solver_macs(n), n * n)

    spans = []  # (worker, stage, block, t0, t1, words)

    def emit(w, stage, blk, t0, dur, words=0):
        spans.append((w, stage, blk, t0, t0 + dur, words))
        return t0 + dur

    # SBR: owner phases in column order
    t = 0.0
    sbr_done = []
    for i in range(W):
        t = emit(i, "SBR", i, t, d_sbr[i], words_sbr[i])
        sbr_done.append(t)
    # relayed chase
    chase_start, chase_done = [], []
    ready = sbr_done[-1] if seq else 0.0
    for i in range(W):
        t0 = max(sbr_done[i], ready)
        ready = emit(i, "BC", i, t0, d_bc[i], words_bc[i])
        chase_start.append(t0)
        chase_done.append(ready)
        if ledger is not None and i < W - 1:
            ledger.record(i, i + 1, "BC", 2 * b * b)
    gathered = chase_done[-1]
    solved = emit(HOST, "Solver", 0, gathered, d_solve, n * n)
    # basis generation (SBR-Back)
    gen_done = []
    for i in range(W):
        if seq:
            if d_gen[i] > 0:
                emit(i, "SBR-Back", i, gathered, d_gen[i])
            gen_done.append(gathered + d_gen[i])
            continue
        first = min(max(chase_start[i] - sbr_done[i], 0.0), d_gen[i])
        if first > 0:
            emit(i, "SBR-Back", i, sbr_done[i], first)
        rest = d_gen[i] - first
        if rest > 0:
            gen_done.append(emit(i, "SBR-Back", i, chase_done[i], rest))
        else:
            gen_done.append(sbr_done[i] + d_gen[i])
    # BC-Back and the final multiply
    if seq:
        t_bb = max(gen_done + [solved])
        bb_done = [emit(i, "BC-Back", i, t_bb, d_bb[i]) for i in range(W)]
        t_fm = max(bb_done)
        ends = [emit(i, "FinalMultiply", i, t_fm, d_fm[i], rows[i] * n) for i in range(W)]
    else:
        bb_done = [emit(i, "BC-Back", i, max(gen_done[i], gathered), d_bb[i]) for i in range(W)]
        ends = [emit(i, "FinalMultiply", i, max(bb_done[i], solved), d_fm[i], rows[i] * n)
                for i in range(W)]
    events = sorted((TraceEvent(w, st, blk, round(t0 * SIM_SCALE), round(t1 * SIM_SCALE), wd)
                     for w, st, blk, t0, t1, wd in spans),
                    key=lambda e: (e.t_start, e.t_end, e.worker, e.stage))
    return events, max(ends)


def fit_b200_seconds_from_bench(path: str) -> dict:
    """Stage seconds from a bench.py JSON line (roofline.stage_ms), for b200_model()."""
    with open(path) as fh:
        line = [x for x in fh if x.strip().startswith("{")][-1]
    d = json.loads(line)
    ms = d["roofline"]["stage_ms"]
    out = dict(B200_STAGE_SECONDS)
    out.update({"n": d["config"]["n"], "b": d["config"]["b"], "SBR": ms["sbr"] / 1e3,
                "BC": ms["bc"] / 1e3, "Solver": ms["solver"] / 1e3,
                "BC-Back": ms["bc_back"] / 1e3})
    return out


__all__ = ["CostModel", "unit_model", "calibrated_model", "b200_model", "load_model", "simulate",
           "SIM_SCALE", "sbr_macs_for_range", "sbr_words_for_range", "bc_macs_for_range",
           "sbr_back_macs", "bc_back_macs", "solver_macs", "final_macs"]
