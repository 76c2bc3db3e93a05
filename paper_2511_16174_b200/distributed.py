"""Multi-GPU pipelined EVD over torch.distributed: one process per GPU (torchrun).

`run_distributed(a, cfg)` on CUDA is the production path: every rank calls the C++ per-rank
orchestrator `pevd_dist_syevd` (csrc/dist.cu) over an NCCL communicator of its own (created
from a unique id that rank 0 shares through the process group).  The protocol (restating
pipeline.py:170-508, the paper's blockwise column distribution):

* SBR (pipeline.py:198-302): rank w owns columns [c0w, c1w) with all n rows.  Per round the
  straddling pieces of a panel are all-gathered, its owner factors it and broadcasts
  [W | Y | T | R]; every rank forms its rows of A W by symmetry and the row blocks are
  all-gathered; every rank updates its own columns (double-blocked, 16 panels per group).
* BC (pipeline.py:306-363): band pieces to rank 0, then the relay: rank w chases the sweeps of
  its columns down the remaining band (bulge.py:348-385) and sends the 2b x b overlap block and
  the band tail to rank w + 1; the tridiagonal pieces and the reflector sets are all-gathered.
* Solver: every rank runs the device divide and conquer (only its back columns of Q_d in
  conventional order); eigenvalues only by bisection.
* Back transformation (pipeline.py:335-420): rows (pipelined / sequential) or columns
  (conventional) of back_plan_sizes; Q slabs are all-gathered on request.

`run_distributed(a, cfg, ops=...)` with a compute object (tests/cpu_ops.py) runs the SAME
message schedule in Python, host-side, so the protocol and its measured ledger are testable
under gloo on CPU: every message either path sends is booked under the same (src, dst, stage,
words), and `schedule.protocol_ledger` states them in closed form.
"""
from __future__ import annotations

import time

import numpy as np
import torch
import torch.distributed as dist

from .core import EigenResult, SymmetricMatrix
from .messaging import BROADCAST, HOST, CommLedger, TraceLog
from .schedule import back_plan_sizes, partition, round_schedule


# ----------------------------------------------------------------------------------------------
# compute interface


# ----------------------------------------------------------------------------------------------
# helpers


def _staged(group, t):
    """gloo moves CPU tensors only: stage CUDA tensors through the host (NCCL uses them as is)."""
    return t.is_cuda and dist.get_backend(group) == "gloo"


def _send(t, dst, group):
    dist.send(t.cpu() if _staged(group, t) else t, dst=dst, group=group)


def _recv(t, src, group):
    if _staged(group, t):
        h = torch.empty(t.shape, dtype=t.dtype)
        dist.recv(h, src=src, group=group)
        t.copy_(h)
    else:
        dist.recv(t, src=src, group=group)


def _p2p(t, src, dst, group):
    """Point to point src -> dst; returns the received tensor on dst (t elsewhere)."""
    rank = dist.get_rank(group)
    if rank == src:
        _send(t.contiguous(), dst, group)
    elif rank == dst:
        _recv(t, src, group)
    return t


def _bcast(t, src, group):
    if _staged(group, t):
        h = t.cpu()
        dist.broadcast(h, src=src, group=group)
        t.copy_(h)
    else:
        dist.broadcast(t, src=src, group=group)


def _allgather_uneven(t: torch.Tensor, counts, group, dim0_extra):
    """All-gather tensors whose first dimension differs per rank (pads to the max)."""
    G = len(counts)
    mx = max(max(counts), 1)
    staged = _staged(group, t)
    dev = torch.device("cpu") if staged else t.device
    buf = torch.zeros((mx,) + tuple(dim0_extra), dtype=t.dtype, device=dev)
    if t.shape[0]:
        buf[: t.shape[0]] = t.to(dev)
    outs = [torch.empty_like(buf) for _ in range(G)]
    dist.all_gather(outs, buf, group=group)
    res = torch.cat([outs[r][: counts[r]] for r in range(G)], dim=0)
    return res.to(t.device) if staged else res


SBR_BACK_AGG = 32  # panels per aggregated SBR-Back block reflector (as the single-GPU path)
SBR_NBB = 16       # panels per double-blocked SBR group (rank-2 * 16 * b trailing updates)


def _aggregate(ops, group, n):
    """One block reflector I - Y T Y^T = H_x0 ... H_x1 for consecutive panels (LAPACK larft
    'F', merged panel by panel): Y is the m0 x K staircase of the panels' Y (zero above each
    panel's first row), T_new = [[T, -T (Y^T Y_x) T_x], [0, T_x]].  Returns (t0, Y, T) as
    column-major device tensors."""
    t0 = group[0][2]
    m0 = n - t0
    K = sum(pw for _, pw, _, _, _ in group)
    Y = ops.zeros(m0, K)
    off = 0
    T = None
    for (c0, pw, tx, Yx, Tx) in group:
        Y[off:off + pw, tx - t0:] = Yx
        if T is None:
            T = Tx.clone()
        else:
            G = ops.zeros(off, pw)
            ops.gemm(Y[:off], Y[off:off + pw], G, ta=True)   # Y_prev^T Y_x
            Tg = ops.zeros(off, pw)
            ops.gemm(T, G, Tg)                                # T G
            T12 = ops.zeros(off, pw)
            ops.gemm(Tg, Tx, T12, alpha=-1.0)                 # -T G T_x
            Tn = ops.zeros(off + pw, off + pw)
            Tn[:off, :off] = T
            Tn[off:, :off] = T12
            Tn[off:, off:] = Tx
            T = Tn
        off += pw
    return t0, Y, T


# ----------------------------------------------------------------------------------------------
# production: the C++ per-rank orchestrator over NCCL


_COMMS: dict = {}


def nccl_comm(group=None):
    """This rank's NCCL communicator for pevd_dist_syevd (created once per process group from a
    unique id that rank 0 shares through the group)."""
    import ctypes
    from . import _lib
    L = _lib.load()
    rank, G = dist.get_rank(group), dist.get_world_size(group)
    key = (id(group), rank, G, torch.cuda.current_device())
    if key not in _COMMS:
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            _lib.check(L.pevd_nccl_unique_id(uid), "nccl unique id")
        box = [bytes(uid.raw)]
        dist.broadcast_object_list(box, src=0, group=group)
        h = ctypes.c_void_p()
        _lib.check(L.pevd_comm_nccl_create(rank, G, box[0], ctypes.byref(h)), "nccl comm")
        _COMMS[key] = h
    return _COMMS[key]


def _gather_outputs(st, group):
    """Every rank's events / messages / flops, merged into the run's TraceEvents, measured
    CommLedger and executed FlopCounter (the same on every rank)."""
    from . import _lib
    mine = {"t0": float(st.t0_mono_ns),
            "events": [(e.worker, e.stage, e.block, e.t_start_ms, e.t_end_ms, e.words)
                       for e in st.events[:min(int(st.n_events), int(st.events_cap))]],
            "msgs": [(m.src, m.dst, m.stage, m.words)
                     for m in st.msgs[:min(int(st.n_msgs), int(st.msgs_cap))]],
            "flops": list(st.stages.flops)}
    G = dist.get_world_size(group)
    allp = [None] * G
    dist.all_gather_object(allp, mine, group=group)
    from .core import FlopCounter
    trace, ledger, counter = TraceLog(), CommLedger(), FlopCounter()
    for p in allp:
        for (w, sg, blk, t0, t1, words) in p["events"]:
            trace.add(w, _lib.TRACE_STAGES[sg], blk, int(round(p["t0"] + t0 * 1e6)),
                      int(round(p["t0"] + t1 * 1e6)), words)
        for (src, dst, sg, words) in p["msgs"]:
            ledger.record(src, dst, _lib.LEDGER_STAGES[sg], words)
        for k, name in enumerate(_lib.FLOP_STAGES):
            if p["flops"][k] > 0:
                counter.add(name, int(round(p["flops"][k] / 2)))
    return trace, ledger, counter


def _run_device(a, cfg, group, n, gather_q):
    """pevd_dist_syevd on this rank's GPU (csrc/dist.cu) over NCCL."""
    import ctypes
    from . import _lib
    from .pipeline import back_ranges
    torch_ = _lib.require_cuda()
    L = _lib.load()
    rank, G = dist.get_rank(group), dist.get_world_size(group)
    if callable(a):
        dense = None
        assert n is not None
    else:
        dense = a.data if isinstance(a, SymmetricMatrix) else \
            SymmetricMatrix.from_dense(np.asarray(a, dtype=np.float64)).data
        n = dense.shape[0]
    b = min(cfg.b, n - 1)
    if b > 64:
        raise ValueError(f"bandwidth b={b} > 64 is not supported by the device kernels")
    cols = partition(n, G)
    backs = back_ranges(n, G, cfg.back_skew)
    c0w, c1w = cols[rank]
    r0, r1 = backs[rank]
    dev = torch_.device("cuda", torch_.cuda.current_device())
    if dense is None:
        blk = a(c0w, c1w)              # (w, n): column-major n x w
    else:
        blk = torch_.from_numpy(np.ascontiguousarray(dense[:, c0w:c1w].T)).to(dev)
    lam = torch_.empty(n, dtype=torch_.float64, device=dev)
    nb = r1 - r0
    qpart = torch_.empty((max(nb, 1), n), dtype=torch_.float64, device=dev) \
        if cfg.want_vectors else None
    col_lo = (ctypes.c_int64 * (G + 1))(*([lo for lo, _ in cols] + [n]))
    back_lo = (ctypes.c_int64 * (G + 1))(*([lo for lo, _ in backs] + [n]))
    st = _lib.new_dist_stats()
    comm = nccl_comm(group)
    P = ctypes.c_void_p
    rc = L.pevd_dist_syevd(comm, n, b, P(blk.data_ptr()), blk.stride(0), col_lo, back_lo,
                           P(lam.data_ptr()), P(qpart.data_ptr()) if qpart is not None else None,
                           n, int(cfg.want_vectors), _lib.ORDER_CODES[cfg.order],
                           P(torch_.cuda.current_stream().cuda_stream), ctypes.byref(st))
    if rc == _lib.PEVD_ERR_CONVERGE:
        raise RuntimeError(L.pevd_last_error().decode())
    _lib.check(rc, f"rank {rank}: pevd_dist_syevd")
    trace, ledger, counter = _gather_outputs(st, group)
    info = {"counter": counter, "stats": st, "cols": (c0w, c1w), "back": (r0, r1),
            "q_part": qpart}
    res = EigenResult(lam=lam.cpu().numpy())
    if cfg.want_vectors and gather_q:
        # (n x nb column-major slabs: Fortran-order columns in conventional order, C-order rows
        #  otherwise) all-gathered over the NCCL process group
        sizes = [hi - lo for lo, hi in backs]
        full = _allgather_uneven(qpart[:nb], sizes, group, (n,))
        for w in range(G):
            ledger.record(w, HOST, "Result", sizes[w] * n)
        qh = full.cpu().numpy()
        res = EigenResult(lam=res.lam, Q=np.asfortranarray(qh.T) if cfg.order == "conventional"
                          else np.ascontiguousarray(qh), vectors_computed=True)
    return res, trace.events(), ledger, info


def run_distributed(a, cfg, ops=None, group=None, n=None, gather_q=True):
    """Blockwise multi-process EVD.

    `a` is either the full matrix (every rank passes the same one; validated like the reference)
    or, for device-resident runs, a callable ``a(c0, c1)`` returning this rank's column block as
    a column-major device tensor of shape (c1 - c0, n) (then `n` must be given).  Every rank gets
    the eigenvalues; with gather_q the full Q too.

    ops=None: the production path on this rank's GPU (csrc/dist.cu over NCCL).  With a compute
    object (tests/cpu_ops.py) the same protocol runs host-side in Python (gloo, CPU tests).

    Returns (EigenResult, events, ledger, info dict)."""
    if ops is None:
        return _run_device(a, cfg, group, n, gather_q)

    rank = dist.get_rank(group)
    G = dist.get_world_size(group)
    if callable(a):
        dense = None
        assert n is not None
    else:
        dense = a.data if isinstance(a, SymmetricMatrix) else \
            SymmetricMatrix.from_dense(np.asarray(a, dtype=np.float64)).data
        n = dense.shape[0]
    ranges = partition(n, G)
    b = min(cfg.b, n - 1) if n > 1 else 0
    c0w, c1w = ranges[rank]
    ledger = CommLedger()
    trace = TraceLog()
    t_base = time.perf_counter_ns()

    def now():  # stage boundaries wait for the device, so the trace spans are device time
        if torch.cuda.is_available() and torch.cuda.is_initialized():
            torch.cuda.synchronize()
        return time.perf_counter_ns() - t_base

    def owner_of(col):
        for x, (lo, hi) in enumerate(ranges):
            if lo <= col < hi:
                return x
        raise AssertionError(col)

    # own column block, all rows: tensor (width, n) = column-major n x width
    blk = a(c0w, c1w) if dense is None else ops.from_host(dense[:, c0w:c1w])
    panels = []  # (c0, pw, t0, Y (pw, m) col-major, T (pw, pw))
    t_sbr0 = now()

    sbr_span = [None, None]   # the rounds this rank owns (its trace SBR event)

    def factor(c0, pw, t0):
        """The panel's straddling pieces are all-gathered, its owner factors it and broadcasts
        [W | Y | T | R] (booked as the reference books (W, Y), pipeline.py:236, plus T, R);
        every rank owning panel columns writes [R; 0] into them.  Returns (Y, W, T)."""
        m = n - t0
        owner = owner_of(c0)
        if rank == owner and sbr_span[0] is None:
            sbr_span[0] = now()
        ov = [max(0, min(c0 + pw, ranges[x][1]) - max(c0, ranges[x][0])) for x in range(G)]
        plo, phi = max(c0, c0w), min(c0 + pw, c1w)
        if ov[owner] < pw:  # straddling panel
            for x in range(G):
                if ov[x]:
                    ledger.record(x, BROADCAST, "SBR-panel", ov[x] * m)
            mine = blk[plo - c0w: phi - c0w, t0:] if plo < phi else \
                torch.zeros((0, m), dtype=torch.float64, device=blk.device)
            P = _allgather_uneven(mine.contiguous(), ov, group, (m,))
        elif rank == owner:
            P = blk[c0 - c0w: c0 + pw - c0w, t0:]
        buf = torch.empty(2 * m * pw + 2 * pw * pw, dtype=torch.float64, device=blk.device)
        if rank == owner:
            R, Y, T = ops.panel_qr(P.contiguous() if ov[owner] < pw else P.clone())
            W = ops.zeros(m, pw)
            ops.gemm(Y, T, W)
            buf[: m * pw] = W.reshape(-1)
            buf[m * pw: 2 * m * pw] = Y.reshape(-1)
            buf[2 * m * pw: 2 * m * pw + pw * pw] = T.reshape(-1)
            buf[2 * m * pw + pw * pw:] = R.reshape(-1)
        ledger.record(owner, BROADCAST, "SBR", 2 * m * pw)        # every rank books every message
        ledger.record(owner, BROADCAST, "SBR-panel", 2 * pw * pw)
        _bcast(buf, owner, group)
        W = buf[: m * pw].reshape(pw, m)
        Y = buf[m * pw: 2 * m * pw].reshape(pw, m)
        T = buf[2 * m * pw: 2 * m * pw + pw * pw].reshape(pw, pw)
        R = buf[2 * m * pw + pw * pw:].reshape(pw, pw)
        if plo < phi:
            Rfull = torch.zeros((pw, m), dtype=torch.float64, device=blk.device)
            Rfull[:, :pw] = R  # panel rows t0.. become [R; 0]
            blk[plo - c0w: phi - c0w, t0:] = Rfull[plo - c0: phi - c0]
        if rank == owner:
            sbr_span[1] = now()
        return Y, W, T

    def form_z(t0, pw, Y, W, corr=None):
        """A W from our columns by symmetry (C5; `corr` subtracts the block's pending
        contribution from our rows), all-gathered, then Z = AW - 1/2 Y (W^T AW)."""
        rlo = max(t0, c0w)
        counts = [max(0, ranges[x][1] - max(t0, ranges[x][0])) for x in range(G)]
        if rlo < c1w:
            cols = blk[rlo - c0w:, t0:]            # (c, m): column-major m x c
            piece_cm = ops.zeros(c1w - rlo, pw)     # (pw, c): column-major c x pw
            ops.gemm(cols, W, piece_cm, ta=True)    # cols^T W
            if corr is not None:
                corr(piece_cm, rlo)
            piece = piece_cm.t().contiguous()       # (c, pw): row-major rows of AW
        else:
            piece = torch.zeros((0, pw), dtype=torch.float64, device=blk.device)
        for x in range(G):
            if counts[x] > 0:
                ledger.record(x, BROADCAST, "SBR", counts[x] * pw)
        AW = _allgather_uneven(piece, counts, group, (pw,)).t().contiguous()  # col-major m x pw
        M = ops.zeros(pw, pw)
        ops.gemm(W, AW, M, ta=True)
        Z = AW.clone()
        ops.gemm(Y, M, Z, alpha=-0.5, beta=1.0)
        return Z

    sched = round_schedule(n, b)
    nrounds = len(sched)
    x = 0
    while x < nrounds:
        c0, pw, t0 = sched[x]
        if pw < b:
            # ---- the ragged last round, one panel (sbr.py:175-182) ----
            Y, W, T = factor(c0, pw, t0)
            Z = form_z(t0, pw, Y, W)
            rlo = max(t0, c0w)
            if rlo < c1w:   # two-sided update of our columns (rows t0..n)
                zlo = rlo - t0
                C = blk[rlo - c0w:, t0:]
                ops.gemm(Y, Z[:, zlo:zlo + (c1w - rlo)], C, alpha=-1.0, beta=1.0, tb=True)
                ops.gemm(Z, Y[:, zlo:zlo + (c1w - rlo)], C, alpha=-1.0, beta=1.0, tb=True)
            klo, khi = max(c0 + pw, c0w), min(t0, c1w)   # coupling columns get Q^T
            if klo < khi:
                cp = blk[klo - c0w: khi - c0w, t0:]
                tmp = ops.zeros(pw, khi - klo)
                ops.gemm(W, cp, tmp, ta=True)
                ops.gemm(Y, tmp, cp, alpha=-1.0, beta=1.0)
            panels.append((c0, pw, t0, Y, T))
            x += 1
            continue
        # ---- a double-blocked group of nbl full panels (as the single-GPU SBR):
        #      P1 = [Y_0 Z_0 Y_1 Z_1 ...], P2 = [Z_0 Y_0 ...] (block rows from t0); panel i's
        #      columns take the pending updates P1 P2^T just before its QR, A W_i is corrected by
        #      -P1 (P2^T W_i), and our trailing columns get ONE rank-2K update at the end
        nbl = 1
        while nbl < SBR_NBB and x + nbl < nrounds and sched[x + nbl][1] == b:
            nbl += 1
        m0 = n - t0
        K = nbl * b
        P1 = ops.zeros(m0, 2 * K)
        P2 = ops.zeros(m0, 2 * K)
        for i in range(nbl):
            ci, _, ti = sched[x + i]
            ri = i * b
            if i:
                lo, hi = max(ci, c0w), min(ci + b, c1w)
                if lo < hi:
                    ops.gemm(P1[: 2 * ri, ri - b:], P2[: 2 * ri, lo - t0: hi - t0],
                             blk[lo - c0w: hi - c0w, ci:], alpha=-1.0, beta=1.0, tb=True)
            Y, W, T = factor(ci, b, ti)
            corr = None
            if i:
                tv = ops.zeros(2 * ri, b)
                ops.gemm(P2[: 2 * ri, ri:], W, tv, ta=True)     # P2^T W_i

                def corr(piece_cm, rlo, tv=tv, ri=ri):
                    ops.gemm(P1[: 2 * ri, rlo - t0: c1w - t0], tv, piece_cm, alpha=-1.0,
                             beta=1.0)
            Z = form_z(ti, b, Y, W, corr)
            P1[2 * ri: 2 * ri + b, ri:] = Y
            P1[2 * ri + b: 2 * ri + 2 * b, ri:] = Z
            P2[2 * ri: 2 * ri + b, ri:] = Z
            P2[2 * ri + b: 2 * ri + 2 * b, ri:] = Y
            panels.append((ci, b, ti, Y, T))
        ru = (nbl - 1) * b
        tl = t0 + ru
        lo = max(tl, c0w)
        if lo < c1w:
            ops.gemm(P1[:, ru:], P2[:, lo - t0: c1w - t0], blk[lo - c0w:, tl:], alpha=-1.0,
                     beta=1.0, tb=True)
        x += nbl
    if sbr_span[0] is not None:
        trace.add(rank, "SBR", rank, sbr_span[0], sbr_span[1])

    # ---- band pieces to rank 0 (BandStage) ----
    width = c1w - c0w
    own_bands = torch.zeros((width, b + 1), dtype=torch.float64, device=blk.device)
    for d in range(b + 1):
        nv = min(width, n - d - c0w)
        if nv > 0:
            j = torch.arange(nv, device=blk.device)
            own_bands[:nv, d] = blk[j, c0w + d + j]
    counts = [hi - lo for lo, hi in ranges]
    for w in range(1, G):
        ledger.record(w, 0, "BandStage", (b + 1) * counts[w])
    bands_rows = _allgather_uneven(own_bands, counts, group, (b + 1,))  # (n, b+1)
    bands = bands_rows.t().contiguous()                                # (b+1, n)
    # ---- the relayed chase (bulge.py:348-385): rank x chases the sweeps of its columns down
    #      the remaining band and hands the overlap block and the tail to rank x + 1 ----
    tail = bands if rank == 0 else None
    parts = None
    for x in range(G):
        c0x = ranges[x][0]
        last = x == G - 1
        pend = n if last else ranges[x + 1][0]
        mr = n - pend
        bwo = min(2 * b, max(mr - 1, 0))
        if rank == x:
            t_bc = now()
            parts = ops.bc_partition(tail, b, c0x, pend, n)
            trace.add(rank, "BC", rank, t_bc, now())
        if not last:
            ledger.record(x, x + 1, "BC", 2 * b * b)
            ledger.record(x, x + 1, "BandStage", (bwo + 1) * mr)
            shape = (bwo + 1, mr)
            t = parts["tail"] if rank == x else torch.empty(shape, dtype=torch.float64)
            t = _p2p(t, x, x + 1, group)
            if rank == x + 1:
                tail = t
    # tridiagonal pieces and reflector sets to every rank
    dcnt = [(n if x == G - 1 else ranges[x + 1][0]) - ranges[x][0] for x in range(G)]
    ecnt = [min(ranges[x][0] + dcnt[x], n - 1) - ranges[x][0] for x in range(G)]
    for x in range(G):
        ledger.record(x, BROADCAST, "Gather", dcnt[x])
        ledger.record(x, BROADCAST, "Gather", ecnt[x])
    d = _allgather_uneven(torch.as_tensor(parts["d"]), dcnt, group, ()).numpy()
    e = _allgather_uneven(torch.as_tensor(parts["e"]), ecnt, group, ()).numpy()
    refl = None
    if cfg.want_vectors:
        sets = [None] * G
        dist.all_gather_object(sets, parts["refl"], group=group)
        vld = ((b + 7) // 8) * 8
        for x in range(G):
            ledger.record(x, BROADCAST, "U-gather", len(sets[x]["tau"]) * (1 + vld))
        refl = ops.merge_reflectors(sets)
    d = torch.as_tensor(d)
    e = torch.as_tensor(e)
    # ---- solver ----
    sizes = back_plan_sizes(n, G, cfg.back_skew)
    bounds = np.cumsum([0] + sizes)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    t_s = now()
    # (conventional order: each rank forms only its own back columns of Q_d)
    if cfg.order == "conventional" and cfg.want_vectors:
        lam, Qd = ops.stedc(d, e, cols=(r0, r1))
    else:
        lam, Qd = ops.stedc(d, e)
    trace.add(rank, "Solver", rank, t_s, now())
    if not cfg.want_vectors:
        return EigenResult(lam=lam), trace.events(), ledger, {}
    if cfg.order == "conventional":
        # ---- conventional order by columns: Q[:, ours] = Q_s Q_b Q_d[:, ours].  Every rank
        #      already holds Q_d, the bulge reflectors and the SBR panels, so the column blocks
        #      are independent: no Q_d / U broadcasts, no final GEMM (pipeline.py:367-387) ----
        t_bb = now()
        X = Qd[r0:r1].clone()                         # column-major n x (r1 - r0)
        X = ops.bc_back_left(n, b, refl, None, X)     # Q_b X
        trace.add(rank, "BC-Back", rank, t_bb, now())
        t_sb = now()
        groups = [panels[g0:g0 + SBR_BACK_AGG] for g0 in range(0, len(panels), SBR_BACK_AGG)]
        for grp in reversed(groups):                  # Q_s X = H_0 (H_1 (... X))
            t0, Yg, Tg = _aggregate(ops, grp, n)
            K = Tg.shape[0]
            X2 = X[:, t0:]                            # rows t0.. of our columns
            P1 = ops.zeros(K, r1 - r0)
            ops.gemm(Yg, X2, P1, ta=True)             # Y^T X
            P2 = ops.zeros(K, r1 - r0)
            ops.gemm(Tg, P1, P2)                      # T (Y^T X)
            ops.gemm(Yg, P2, X2, alpha=-1.0, beta=1.0)  # X -= Y T Y^T X
        trace.add(rank, "SBR-Back", rank, t_sb, now())
        if not gather_q:
            return (EigenResult(lam=lam), trace.events(), ledger,
                    {"cols": (r0, r1), "q_cols": X})
        Qc = _allgather_uneven(X, sizes, group, (n,))    # (n cols, n rows): column-major Q
        for w in range(G):
            ledger.record(w, HOST, "Result", sizes[w] * n)
        return (EigenResult(lam=lam, Q=np.asfortranarray(Qc.cpu().numpy().T),
                            vectors_computed=True),
                trace.events(), ledger, {"cols": (r0, r1)})
    # ---- back transformation of our rows ----
    t_sb = now()
    Mt = ops.zeros(r1 - r0, n)               # column-major (r x n): rows r0..r1 of I
    ir = torch.arange(r1 - r0, device=Mt.device)
    Mt[r0 + ir, ir] = 1.0
    for g0 in range(0, len(panels), SBR_BACK_AGG):    # M <- M (I - Y T Y^T), creation order
        t0, Yg, Tg = _aggregate(ops, panels[g0:g0 + SBR_BACK_AGG], n)
        K = Tg.shape[0]
        Ms = Mt[t0:]                          # column-major r x m
        P1 = ops.zeros(r1 - r0, K)
        ops.gemm(Ms, Yg, P1)                  # M Y
        P2 = ops.zeros(r1 - r0, K)
        ops.gemm(P1, Tg, P2)                  # (M Y) T
        ops.gemm(P2, Yg, Ms, alpha=-1.0, beta=1.0, tb=True)  # -= (M Y T) Y^T
    trace.add(HOST if cfg.order == "pipelined" else rank, "SBR-Back", rank, t_sb, now())
    t_bb = now()
    Msb = ops.bc_back_right(n, b, refl, None, Mt)   # rows of Q_s Q_b (in place)
    trace.add(HOST if cfg.order == "pipelined" else rank, "BC-Back", rank, t_bb, now())
    dist.barrier(group)  # Q_d complete everywhere before any final multiply (dist.cu does the same)
    t_f = now()
    Qrows_t = ops.zeros(r1 - r0, n)
    ops.gemm(Msb, Qd, Qrows_t)
    trace.add(rank, "FinalMultiply", rank, t_f, now())
    if not gather_q:
        return (EigenResult(lam=lam), trace.events(), ledger,
                {"rows": (r0, r1), "q_rows": Qrows_t})
    Qrows = Qrows_t.t().contiguous()                          # (r, n) row-major
    Q = _allgather_uneven(Qrows, sizes, group, (n,))          # (n, n) row-major == C order
    for w in range(G):
        ledger.record(w, HOST, "Result", sizes[w] * n)
    return (EigenResult(lam=lam, Q=np.ascontiguousarray(Q.cpu().numpy()), vectors_computed=True),
            trace.events(), ledger, {"rows": (r0, r1)})
