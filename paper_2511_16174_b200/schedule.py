"""Host-side scheduling arithmetic of the pipelined EVD (no device work).

Restates the reference's partition / round / back-plan rules and the analytic communication
formulas (pipeevd/schedule.py:21-79, sbr.py:54-66, backtrans.py:62-121) so the distributed
driver and the ledger use exactly the reference's numbers.
"""
from __future__ import annotations

import math


def partition(n: int, workers: int) -> list[tuple[int, int]]:
    """Contiguous column ranges, remainder to the front (schedule.py:21-33)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if workers > n:
        raise ValueError(f"cannot split {n} columns over {workers} workers")
    base, rem = divmod(n, workers)
    out, at = [], 0
    for w in range(workers):
        size = base + (1 if w < rem else 0)
        out.append((at, at + size))
        at += size
    return out


def round_schedule(n: int, b: int) -> list[tuple[int, int, int]]:
    """(col_start, panel_width, trailing_start) per SBR round (sbr.py:54-66)."""
    out, c0 = [], 0
    while c0 < n - b:
        out.append((c0, min(b, n - b - c0), c0 + b))
        c0 += b
    return out


def comm_triangular_words(n: int, b: int) -> float:
    """Words if trailing triangles were shipped every round (schedule.py:36-50)."""
    if n < 1 or b < 1:
        raise ValueError("n and b must be positive")
    total, i = 0, 1
    while n - i * b > 0:
        total += (n - i * b) ** 2
        i += 1
    return total / 2.0


def comm_broadcast_words(n: int, b: int) -> int:
    """Words broadcast per reduction, 3 (n - i b) b summed over rounds (schedule.py:53-68)."""
    if n < 1 or b < 1:
        raise ValueError("n and b must be positive")
    return sum(3 * (n - c0 - b) * pw for c0, pw, _ in round_schedule(n, b))


def crossover_bandwidth(p: float, q: float) -> int:
    """Largest bandwidth b with b < 4p/q (schedule.py:71-79)."""
    if p <= 0 or q <= 0:
        raise ValueError("rates must be positive")
    return math.ceil(4.0 * p / q) - 1


class BackPlan:
    """Per-worker row block sizes of the back transform (backtrans.py:30-59)."""

    def __init__(self, sizes, base):
        self.sizes = [int(s) for s in sizes]
        self.base = int(base)
        if any(s < 1 for s in self.sizes):
            raise ValueError("empty back-transform block")
        if any(self.sizes[i] < self.sizes[i + 1] for i in range(len(self.sizes) - 1)):
            raise ValueError("block sizes must be non-increasing")
        for s in self.sizes:
            if 20 * abs(s - self.base) > self.base:
                raise ValueError(f"block size {s} deviates more than 5% from base {self.base}")

    @property
    def n(self) -> int:
        return sum(self.sizes)

    def column_ranges(self):
        out, at = [], 0
        for s in self.sizes:
            out.append((at, at + s))
            at += s
        return out


def make_back_plan(n: int, workers: int, base: int, skew: float) -> BackPlan:
    """Ramped sizes round(base (1 + skew (1 - 2i/(w-1)))) repaired to sum n inside the 5%
    corridor (backtrans.py:62-105)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if not 0.0 <= skew <= 0.05:
        raise ValueError(f"skew {skew} outside [0, 0.05]")
    if base < 1:
        raise ValueError("base must be >= 1")
    if workers == 1:
        if 20 * abs(n - base) > base:
            raise ValueError(f"cannot split {n} columns into 1 block of base {base} within 5%")
        return BackPlan([n], base)
    ideal = [base * (1.0 + skew * (1.0 - 2.0 * i / (workers - 1))) for i in range(workers)]
    sizes = [round(x) for x in ideal]
    for i in range(workers):
        while 20 * abs(sizes[i] - base) > base:
            sizes[i] += 1 if sizes[i] < base else -1
    delta = n - sum(sizes)
    step = 1 if delta > 0 else -1
    for _ in range(abs(delta)):
        best, best_cost = -1, None
        for i in range(workers):
            cand = sizes[i] + step
            if cand >= 1 and 20 * abs(cand - base) <= base:
                cost = abs(cand - ideal[i])
                if best_cost is None or cost < best_cost:
                    best, best_cost = i, cost
        if best < 0:
            raise ValueError(f"cannot split {n} columns into {workers} blocks of base {base} within 5%")
        sizes[best] += step
    sizes.sort(reverse=True)
    return BackPlan(sizes, base)


def back_plan_sizes(n: int, workers: int, skew: float) -> list[int]:
    """Row-block sizes for the back transform, falling back to an even split
    (backtrans.py:108-121)."""
    if not 0.0 <= skew <= 0.05:
        raise ValueError(f"skew {skew} outside [0, 0.05]")
    try:
        return make_back_plan(n, workers, max(1, round(n / workers)), skew).sizes
    except ValueError:
        base, rem = divmod(n, workers)
        return [base + (1 if i < rem else 0) for i in range(workers)]


# ---------------------------------------------------------------------------- MAC formulas
# The FlopCounter contract (core.py:5-6): multiply-adds per stage, matching the reference's
# counted kernels for the operations the device performs.

def sbr_macs(n: int, b: int) -> int:
    """panel QR + form_z + rank-2k (sbr.py:69-152 counters, symmetric mode ~ lower tiles)."""
    tot = 0
    for c0, pw, t0 in round_schedule(n, b):
        m = n - t0
        tot += 2 * m * pw * pw            # panel QR (rank-1 + W)
        tot += m * m * pw + 2 * m * pw * pw  # A W, W^T AW, Y M
        tot += m * (m + 1) * pw           # rank-2k, lower half (2 m^2 pw / 2)
    return tot


def bc_macs(n: int, b: int) -> int:
    """~7 b^2 MACs per chase step (schedule.py:122); exact per-step count of bulge.py:170-252."""
    tot = 0
    for i in range(max(n - 2, 0)):
        j = 0
        while i + 1 + j * b <= n - 2:
            w0 = i + 1 + j * b
            L = min(b, n - w0)
            nleft = 0 if j == 0 else b - 1
            nT = min(w0 + L + b, n) - (w0 + L)
            tot += 2 * L * nleft + 3 * L * L + 3 * L + 2 * L * nT
            j += 1
    return tot


def bc_macs_fast(n: int, b: int) -> int:
    """Closed-form approximation of bc_macs for large n (7 b^2 per reflector)."""
    nref = 0
    j = 0
    while n - 2 - j * b > 0:
        nref += n - 2 - j * b
        j += 1
    return 7 * b * b * nref


def bc_back_macs(n: int, b: int, ncols: int) -> int:
    """2 len m per reflector (backtrans.py:273)."""
    tot = 0
    j = 0
    while n - 2 - j * b > 0:
        for i in range(n - 2 - j * b):
            r0 = i + 1 + j * b
            tot += 2 * min(b, n - r0) * ncols
        j += 1
    return tot


def bc_back_macs_fast(n: int, b: int, ncols: int) -> int:
    nref = 0
    j = 0
    while n - 2 - j * b > 0:
        nref += n - 2 - j * b
        j += 1
    return 2 * b * nref * ncols


# ------------------------------------------------------------------ trace contract
def validate_trace(events, workers: int, ledger=None) -> None:
    """Raise ValueError when a trace breaks the pipeline's dependency contract
    (schedule.py:334-386): no two non-Comm events of one worker overlap; the SBR and BC chains
    run worker after worker; BC-Back starts after every BC event (the reflector gather);
    FinalMultiply starts after the solver; with a ledger, exactly one boundary message per
    neighbouring worker pair in the BC stage."""
    for w in range(workers):
        mine = sorted((e for e in events if e.worker == w and e.stage != "Comm"),
                      key=lambda e: (e.t_start, e.t_end))
        for x, y in zip(mine, mine[1:]):
            if y.t_start < x.t_end:
                raise ValueError(f"worker {w}: {x.stage} [{x.t_start},{x.t_end}) overlaps "
                                 f"{y.stage} [{y.t_start},{y.t_end})")
    for stage in ("SBR", "BC"):
        for w in range(workers - 1):
            left = [e.t_end for e in events if e.stage == stage and e.worker == w]
            right = [e.t_start for e in events if e.stage == stage and e.worker == w + 1]
            if left and right and max(left) > min(right):
                raise ValueError(f"{stage} chain broken between workers {w} and {w + 1}")

    def ends(stage):
        return [e.t_end for e in events if e.stage == stage]

    def starts(stage):
        return [e.t_start for e in events if e.stage == stage]

    if ends("BC") and starts("BC-Back") and min(starts("BC-Back")) < max(ends("BC")):
        raise ValueError(f"BC-Back starts at {min(starts('BC-Back'))} before the reflector "
                         f"gather completes at {max(ends('BC'))}")
    if ends("Solver") and starts("FinalMultiply") and \
            min(starts("FinalMultiply")) < max(ends("Solver")):
        raise ValueError(f"FinalMultiply starts at {min(starts('FinalMultiply'))} before the "
                         f"solver finishes at {max(ends('Solver'))}")
    if ledger is not None and workers > 1:
        for w in range(workers - 1):
            m = ledger.messages(stage="BC", src=w, dst=w + 1)
            if m != 1:
                raise ValueError(f"expected exactly one overlap message from worker {w} to "
                                 f"{w + 1}, ledger has {m}")
        total = ledger.messages(stage="BC")
        if total != workers - 1:
            raise ValueError(f"stray BC-stage messages: {total} total for {workers - 1} "
                             f"boundaries")


def mean_idle_fraction(events, workers: int) -> float:
    """1 - busy / span averaged over the workers, helper lanes excluded (schedule.py:389-402)."""
    spans = [e for e in events if e.stage != "Comm"]
    if not spans:
        return 0.0
    t0 = min(e.t_start for e in spans)
    t1 = max(e.t_end for e in spans)
    if t1 == t0:
        return 0.0
    return sum(1.0 - sum(e.duration for e in spans if e.worker == w) / (t1 - t0)
               for w in range(workers)) / workers


# ------------------------------------------------------------------ the measured protocol
def protocol_ledger(n: int, b: int, workers: int, want_vectors: bool = True,
                    back_skew: float = 0.0, result: bool = True) -> list:
    """Every message of the blockwise protocol (csrc/dist.cu, distributed.py) as
    (src, dst, stage, words), in closed form from the schedule -- the ledger a run measures.
    dst -1 = host, -2 = broadcast (messaging.py).  `result`: the Q slabs gathered to the caller.
      SBR        per round: owner broadcasts (W, Y) 2 m pw (pipeline.py:236); every rank its
                 A W row block (pipeline.py:251-271) -> sum = comm_broadcast_words(n, b)
      SBR-panel  T and R of the factor (2 pw^2); straddling pieces (overlap x m per holder)
      BandStage  band pieces to rank 0; the band tail rank x -> x + 1 ((bw + 1) x rest)
      BC         the 2b x b overlap block rank x -> x + 1 (bulge.py:144-167)
      Gather     each partition's d and e pieces
      U-gather   each partition's reflectors, (1 + pad8(b)) words each
      Result     the Q slab of each worker (n x back block)"""
    G = workers
    if G < 2:
        return []  # one worker moves nothing between devices
    ranges = partition(n, G)
    msgs = []

    def owner(c):
        return next(x for x, (lo, hi) in enumerate(ranges) if lo <= c < hi)

    for c0, pw, t0 in round_schedule(n, b):
        m = n - t0
        o = owner(c0)
        ov = [max(0, min(c0 + pw, hi) - max(c0, lo)) for lo, hi in ranges]
        if ov[o] < pw:
            msgs += [(x, -2, "SBR-panel", ov[x] * m) for x in range(G) if ov[x]]
        msgs.append((o, -2, "SBR", 2 * m * pw))
        msgs.append((o, -2, "SBR-panel", 2 * pw * pw))
        for x, (lo, hi) in enumerate(ranges):
            c = hi - max(t0, lo)
            if c > 0:
                msgs.append((x, -2, "SBR", c * pw))
    for x in range(1, G):
        msgs.append((x, 0, "BandStage", (b + 1) * (ranges[x][1] - ranges[x][0])))
    J = (n - 3) // b + 1 if n >= 3 else 0
    vld = ((b + 7) // 8) * 8
    for x in range(G):
        c0 = ranges[x][0]
        pend = n if x == G - 1 else ranges[x + 1][0]
        if x < G - 1:
            mr = n - pend
            msgs.append((x, x + 1, "BC", 2 * b * b))
            msgs.append((x, x + 1, "BandStage", (min(2 * b, max(mr - 1, 0)) + 1) * mr))
        msgs.append((x, -2, "Gather", pend - c0))
        msgs.append((x, -2, "Gather", min(pend, n - 1) - c0))
        if want_vectors and G > 1:
            npiv = pend - c0
            cnt = sum(max(0, min(npiv, n - c0 - 2 - j * b)) for j in range(J))
            msgs.append((x, -2, "U-gather", cnt * (1 + vld)))
    if want_vectors and result:
        for x, s in enumerate(back_plan_sizes(n, G, back_skew)):
            msgs.append((x, -1, "Result", s * n))
    return [m_ for m_ in msgs if m_[3] > 0]
