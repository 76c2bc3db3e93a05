"""Drop-in `run(a, PipelineConfig)` of the pipelined two-stage FP64 EVD (pipeline.py:57-573).

`run` validates and copies the input exactly like the reference (core.py:65-93,
pipeline.py:511-548), then executes the whole EVD on the GPU through the C ABI
(pevd_syevd_device, include/pevd.h): SBR -> BC -> divide and conquer, with SBR-Back and BC-Back
on a second CUDA stream ("pipelined"), the same stages on one stream ("sequential"), or the
reflectors applied to Q_d from the left ("conventional").  The returned 4-tuple keeps the
reference's contract: EigenResult, time-sorted TraceEvents (device CUDA-event stage times),
CommLedger, FlopCounter (MACs).

Trace lanes: worker 0 is the main stream (SBR, BC, Solver, FinalMultiply); the back-transform
stream (SBR-Back, BC-Back), which overlaps the chase and the solver, is reported as the
concurrent helper lane HOST (-1), the role the reference's host thread plays.

Ledger: one GPU moves no messages; the ledger records the words the reference's blockwise
protocol exchanges between `cfg.workers` devices (pipeline.py:236-502), so analytic checks
(schedule.comm_broadcast_words, 2 b^2 per BC boundary) hold for any worker count.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .core import EigenResult, FlopCounter, SymmetricMatrix
from .messaging import BROADCAST, HOST, CommLedger, TraceLog
from .schedule import (back_plan_sizes, bc_back_macs, bc_back_macs_fast, bc_macs, bc_macs_fast,
                       partition, round_schedule, sbr_macs)

ORDERS = ("pipelined", "sequential", "conventional")


class PipelineError(RuntimeError):
    """A device or stage failed; the message names who and in which stage (pipeline.py:50)."""


@dataclass
class PipelineConfig:
    """Knobs of one run (pipeline.py:57-82)."""

    workers: int
    b: int = 32
    order: str = "pipelined"
    back_skew: float = 0.0
    seed: int | None = None
    trace_path: str | None = None
    want_vectors: bool = True

    def __post_init__(self):
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.b < 1:
            raise ValueError("bandwidth must be >= 1")
        if self.order not in ORDERS:
            raise ValueError(f"order must be one of {ORDERS}, not {self.order!r}")
        if not 0.0 <= self.back_skew <= 0.05:
            raise ValueError(f"back_skew {self.back_skew} outside [0, 0.05]")


def _ledger_for(n: int, b: int, cfg: PipelineConfig, nref: int) -> CommLedger:
    """Words of the blockwise protocol for cfg.workers devices (pipeline.py:236-502)."""
    led = CommLedger()
    W = cfg.workers
    if b < 1:
        return led
    ranges = partition(n, W)
    owner = [next(w for w, (lo, hi) in enumerate(ranges) if lo <= c0 < hi)
             for c0, _, _ in round_schedule(n, b)]
    for idx, (c0, pw, t0) in enumerate(round_schedule(n, b)):
        m = n - t0
        led.record(owner[idx], BROADCAST, "SBR", 2 * m * pw)     # ("wy", idx): W and Y
        for x, (lo, hi) in enumerate(ranges):
            rlo = max(t0, lo)
            if rlo < hi:
                led.record(x, BROADCAST, "SBR", (hi - rlo) * pw)  # ("aw", idx) row block
    for w in range(W):
        led.record(w, HOST, "BandStage", (b + 1) * (ranges[w][1] - ranges[w][0]))
    for w in range(W - 1):
        led.record(w, w + 1, "BC", 2 * b * b)                   # the 2b x b overlap block
    if cfg.want_vectors:
        stride = ((b + 7) // 8) * 8
        led.record(HOST, BROADCAST, "U-gather", 4 * nref + nref + nref * stride)
        if cfg.order != "conventional":
            led.record(HOST, BROADCAST, "Qd", n * n)
    return led


def _macs(n: int, b: int, cfg: PipelineConfig) -> FlopCounter:
    c = FlopCounter()
    if n < 2 or b < 1:
        return c
    c.add("SBR", sbr_macs(n, b))
    c.add("BC", bc_macs(n, b) if n <= 4096 else bc_macs_fast(n, b))
    # D&C merge GEMMs without deflation: sum over levels of (n1^2 + n2^2) s ~ (2/3) n^3 MACs
    c.add("Solver", max(1, (2 * n ** 3) // 3))
    if cfg.want_vectors:
        c.add("SBR-Back", max(1, (2 * n ** 3) // 3))
        c.add("BC-Back", bc_back_macs(n, b, n) if n <= 2048 else bc_back_macs_fast(n, b, n))
        if cfg.order != "conventional":
            c.add("FinalMultiply", n ** 3)
    return c


def run(a, cfg: PipelineConfig):
    """A = Q diag(lam) Q^T on the GPU; returns (EigenResult, events, ledger, counter)."""
    if isinstance(a, SymmetricMatrix):
        dense = a.data
    else:
        dense = SymmetricMatrix.from_dense(np.asarray(a, dtype=np.float64)).data
    n = int(dense.shape[0])
    partition(n, cfg.workers)  # raises ValueError for workers > n (schedule.py:26-27)
    b = min(cfg.b, n - 1) if n > 1 else 0
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1 and n > 2:
        # one process per GPU: the blockwise protocol (distributed.py)
        from .distributed import run_distributed
        from .core import FlopCounter as _FC
        res, events, ledger, _ = run_distributed(dense, cfg)
        if cfg.trace_path:
            log = TraceLog()
            for ev in events:
                log.add(ev.worker, ev.stage, ev.block, ev.t_start, ev.t_end, ev.words)
            log.to_ndjson(cfg.trace_path)
        return res, events, ledger, _macs(n, b, cfg)
    from . import device  # imports torch lazily; fails loudly without CUDA / libpevd.so
    t0 = time.perf_counter_ns()
    try:
        lam, q, st = device.syevd(dense, max(b, 1), cfg.want_vectors, cfg.order)
    except ValueError:
        raise
    except RuntimeError as exc:  # non-convergence keeps the reference's exception type
        if "did not converge" in str(exc):
            raise
        raise PipelineError(f"worker 0 failed during device EVD: {exc!r}") from exc
    trace = TraceLog()
    ns = lambda ms: t0 + int(round(ms * 1e6))  # noqa: E731
    if n > 1:
        trace.add(0, "SBR", 0, ns(st.sbr_ms[0]), ns(st.sbr_ms[1]))
        trace.add(0, "BC", 0, ns(st.bc_ms[0]), ns(st.bc_ms[1]))
        trace.add(0, "Solver", 0, ns(st.solver_ms[0]), ns(st.solver_ms[1]))
        if cfg.want_vectors:
            back = HOST if cfg.order == "pipelined" else 0
            trace.add(back, "SBR-Back", 0, ns(st.sbr_back_ms[0]), ns(st.sbr_back_ms[1]))
            trace.add(back, "BC-Back", 0, ns(st.bc_back_ms[0]), ns(st.bc_back_ms[1]))
            trace.add(0, "FinalMultiply", 0, ns(st.final_ms[0]), ns(st.final_ms[1]))
    nref = int(st.n_reflectors)
    ledger = _ledger_for(n, b, cfg, nref) if n > 1 else CommLedger()
    counter = _macs(n, b, cfg)
    result = EigenResult(lam=lam, Q=q if cfg.want_vectors else None,
                         vectors_computed=bool(cfg.want_vectors))
    if cfg.want_vectors and cfg.order == "conventional":
        result.Q = np.asfortranarray(result.Q)
    elif cfg.want_vectors:
        result.Q = np.ascontiguousarray(result.Q)  # pipeline.py:503 (C order)
    if cfg.trace_path:
        trace.to_ndjson(cfg.trace_path)
    return result, trace.events(), ledger, counter


def run_auto_skew(a, cfg: PipelineConfig):
    """Run once, derive back_skew from the idle gap, run again (pipeline.py:551-573)."""
    first = run(a, cfg)
    busy = [0] * cfg.workers
    t_lo, t_hi = None, 0
    for ev in first[1]:
        if ev.worker < 0 or ev.stage == "Comm":
            continue
        busy[ev.worker] += ev.duration
        t_hi = max(t_hi, ev.t_end)
        t_lo = ev.t_start if t_lo is None else min(t_lo, ev.t_start)
    span = max(1, t_hi - (t_lo or 0))
    idle = [1.0 - bz / span for bz in busy]
    skew = min(0.05, max(0.0, 0.5 * (idle[-1] - idle[0])))
    cfg2 = replace(cfg, back_skew=round(skew, 4))
    return run(a, cfg2) + (cfg2.back_skew,)


def back_rows(n: int, cfg: PipelineConfig):
    """Row blocks of the back transform per worker (pipeline.py:97-102)."""
    sizes = back_plan_sizes(n, cfg.workers, cfg.back_skew)
    out, at = [], 0
    for s in sizes:
        out.append((at, at + s))
        at += s
    return out


__all__ = ["PipelineConfig", "PipelineError", "run", "run_auto_skew", "ORDERS", "_lib"]
