"""Drop-in `run(a, PipelineConfig)` of the pipelined two-stage FP64 EVD (pipeline.py:57-573).

`run` validates and copies the input exactly like the reference (core.py:65-93,
pipeline.py:511-548), then executes the whole EVD on the GPU through the C ABI
(pevd_syevd_device, include/pevd.h): SBR -> BC -> divide and conquer, with SBR-Back and BC-Back
on a second CUDA stream ("pipelined"), the same stages on one stream ("sequential"), or the
reflectors applied to Q_d from the left ("conventional").  The returned 4-tuple keeps the
reference's contract: EigenResult, time-sorted TraceEvents (device CUDA-event stage times),
CommLedger, FlopCounter (MACs).

Workers: workers = 1 runs the fused single-GPU orchestrator.  workers = G > 1 runs the paper's
blockwise protocol over G cooperating devices -- in this process (pevd_syevd_multi: one host
thread per worker, peer-to-peer copies over NVLink; workers map round-robin onto the visible
GPUs, so a 1-GPU box runs G workers on one device) or, under torchrun, one process per GPU over
NCCL (distributed.py).

Trace lanes: a worker's main stream (SBR rounds it owns, its BC partition, Solver,
FinalMultiply; Comm spans on its comm stream); the back-transform stream, which overlaps the
chase and the solver in pipelined order, is the concurrent helper lane HOST (-1), the role the
reference's host thread plays.

Ledger and counter are MEASURED: every message is booked with the words actually handed to the
transport (schedule.protocol_ledger states them in closed form; the SBR words equal
comm_broadcast_words and each BC boundary carries one 2b x b overlap block, as in the
reference), and the FlopCounter holds the executed multiply-adds per stage (PevdStats.flops).
"""
from __future__ import annotations

import time
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .core import EigenResult, FlopCounter, SymmetricMatrix
from .messaging import BROADCAST, HOST, CommLedger, TraceLog
from .schedule import back_plan_sizes, partition

ORDERS = ("pipelined", "sequential", "conventional")
HOST_CHECK_MAX_N = 4096  # above this the input's symmetry check runs on the device


def _cuda_ready() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


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


def dist_outputs(stats, workers: int):
    """TraceEvents, the measured CommLedger and the executed-flop FlopCounter (MACs) of a
    distributed run, from the per-rank PevdDistStats (pevd.h).  Event times are CLOCK_MONOTONIC
    ns (time.perf_counter_ns's clock): each rank's t0 is taken after a barrier of all ranks."""
    trace, ledger, counter = TraceLog(), CommLedger(), FlopCounter()
    for st in stats:
        t0 = float(st.t0_mono_ns)
        for i in range(min(int(st.n_events), int(st.events_cap))):
            e = st.events[i]
            trace.add(e.worker, _lib.TRACE_STAGES[e.stage], e.block,
                      int(round(t0 + e.t_start_ms * 1e6)), int(round(t0 + e.t_end_ms * 1e6)),
                      e.words)
        for i in range(min(int(st.n_msgs), int(st.msgs_cap))):
            m = st.msgs[i]
            ledger.record(m.src, m.dst, _lib.LEDGER_STAGES[m.stage], m.words)
        for k, name in enumerate(_lib.FLOP_STAGES):
            if st.stages.flops[k] > 0:
                counter.add(name, int(round(st.stages.flops[k] / 2)))
    return trace, ledger, counter


def _macs(st) -> FlopCounter:
    """Executed multiply-adds per stage of a single-GPU run (PevdStats.flops / 2)."""
    c = FlopCounter()
    for k, name in enumerate(_lib.FLOP_STAGES):
        if st.flops[k] > 0:
            c.add(name, int(round(st.flops[k] / 2)))
    return c


def back_ranges(n: int, workers: int, back_skew: float):
    """Row (pipelined / sequential) or column (conventional) blocks of the back transform
    (pipeline.py:97-102, backtrans.py:108-121)."""
    sizes = back_plan_sizes(n, workers, back_skew)
    out, at = [], 0
    for s in sizes:
        out.append((at, at + s))
        at += s
    return out


def run(a, cfg: PipelineConfig):
    """A = Q diag(lam) Q^T on the GPU; returns (EigenResult, events, ledger, counter)."""
    device_check = False
    if isinstance(a, SymmetricMatrix):
        dense = a.data
    else:
        arr = np.asarray(a, dtype=np.float64)
        if arr.ndim == 2 and arr.shape[0] == arr.shape[1] and arr.shape[0] > HOST_CHECK_MAX_N \
                and cfg.workers == 1 and _cuda_ready():
            # large inputs: the SymmetricMatrix check (core.py:75-84) runs on the device after the
            # copy the EVD needs anyway, instead of an n^2 host temporary; no host F-order copy
            dense, device_check = arr, True
        else:
            dense = SymmetricMatrix.from_dense(arr).data
    n = int(dense.shape[0])
    partition(n, cfg.workers)  # raises ValueError for workers > n (schedule.py:26-27)
    b = min(cfg.b, n - 1) if n > 1 else 0
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1 and n > 2:
        # one process per GPU (torchrun): every rank runs the C++ per-rank orchestrator over NCCL
        if cfg.workers != dist.get_world_size():
            raise ValueError(f"PipelineConfig.workers={cfg.workers} but the process group has "
                             f"{dist.get_world_size()} ranks (one worker per rank)")
        from .distributed import run_distributed
        res, events, ledger, info = run_distributed(dense, cfg)
        if cfg.trace_path:
            log = TraceLog()
            for ev in events:
                log.add(ev.worker, ev.stage, ev.block, ev.t_start, ev.t_end, ev.words)
            log.to_ndjson(cfg.trace_path)
        return res, events, ledger, info["counter"]
    from . import device  # imports torch lazily; fails loudly without CUDA / libpevd.so
    if cfg.workers > 1 and n >= 3:
        return _run_multi(dense, n, b, cfg, device)
    t0 = time.perf_counter_ns()
    try:
        lam, q, st = device.syevd(dense, max(b, 1), cfg.want_vectors, cfg.order,
                                  check_sym=device_check)
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
            if cfg.order != "conventional":  # conventional order has no final multiply
                trace.add(0, "FinalMultiply", 0, ns(st.final_ms[0]), ns(st.final_ms[1]))
    ledger = CommLedger()  # one GPU: nothing moves between devices
    counter = _macs(st)
    result = EigenResult(lam=lam, Q=q if cfg.want_vectors else None,
                         vectors_computed=bool(cfg.want_vectors))
    # (device.syevd returns Q Fortran-ordered in conventional order, C-ordered otherwise:
    #  pipeline.py:495, 503)
    if cfg.trace_path:
        trace.to_ndjson(cfg.trace_path)
    return result, trace.events(), ledger, counter


def _run_multi(dense, n: int, b: int, cfg: PipelineConfig, device):
    """cfg.workers cooperating devices in this process (pevd_syevd_multi): the blockwise
    protocol with one host thread per worker and peer-to-peer transfers.  Workers map
    round-robin onto the visible GPUs; on a box with fewer GPUs than workers several workers
    share one device (the same protocol and messages, without the extra parallelism)."""
    if b > 64:
        raise ValueError(f"bandwidth b={b} > 64 is not supported by the device kernels")
    cols = partition(n, cfg.workers)
    backs = back_ranges(n, cfg.workers, cfg.back_skew)
    try:
        lam, q, stats = device.syevd_multi(dense, cfg.workers, max(b, 1), cols, backs,
                                           cfg.want_vectors, cfg.order)
    except ValueError:
        raise
    except RuntimeError as exc:
        if "did not converge" in str(exc):
            raise
        raise PipelineError(f"distributed EVD failed: {exc}") from exc
    trace, ledger, counter = dist_outputs(stats, cfg.workers)
    result = EigenResult(lam=lam, Q=q if cfg.want_vectors else None,
                         vectors_computed=bool(cfg.want_vectors))
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
    return back_ranges(n, cfg.workers, cfg.back_skew)


__all__ = ["PipelineConfig", "PipelineError", "run", "run_auto_skew", "ORDERS", "_lib"]
