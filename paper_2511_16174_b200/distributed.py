"""Multi-GPU pipelined EVD: the paper's blockwise column distribution over torch.distributed.

Restates the reference's worker/host protocol (pipeline.py:170-508) for one process per GPU:

* SBR (pipeline.py:198-302): rank w owns columns [c0w, c1w) with all n rows (full storage,
  schedule.py:21-33).  Per round the panel's owner gathers straddling pieces (C2/C3), factors it
  (panel QR on its device), and broadcasts the factor (C4); every rank forms its rows of A W by
  symmetry from its own columns and all-gathers them (C5); every rank then applies the two-sided
  update to its own columns only.  The trailing matrix never moves.
* BC (pipeline.py:306-363): the band is all-gathered (13 MB at n=49152) and every rank runs the
  wavefront chase on its device.  Over NVSwitch this replaces the reference's serial relay of the
  overlap block and the 10 GB reflector all-gather (C7-C10) with one band all-gather; the result
  is bitwise identical on every rank because the chase kernel is deterministic.
* Solver: every rank runs the device divide and conquer (no 19 GB Q_d broadcast, C11).
* Back transformation (pipeline.py:335-420): rank w owns rows back_plan_sizes(...)[w] of Q.  It
  accumulates its rows of Q_s panel by panel (RowAccumulator), applies the bulge reflectors
  (BC-Back, reordered) and multiplies by Q_d; rows are all-gathered at the end (C12).

The compute goes through an `ops` object: `CudaOps` (libpevd.so, production) or a CPU
implementation supplied by the tests (so the protocol runs under gloo without a GPU).  The
ledger records the words the reference's protocol counts (messaging.py:111-167), so its analytic
checks (comm_broadcast_words, 2 b^2 per BC boundary) read the same.
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


class CudaOps:
    """Device compute over the C ABI (column-major matrices as torch tensors of shape (cols, rows)
    on the current CUDA device)."""

    def __init__(self):
        from . import _lib
        self.torch = _lib.require_cuda()
        self.L = _lib.load()
        self._lib = _lib
        self.device = torch.device("cuda", torch.cuda.current_device())

    # -- memory
    def from_host(self, a):  # numpy (rows x cols) -> column-major device tensor
        return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64).T)).to(self.device)

    def to_host(self, t):
        return np.asfortranarray(t.detach().cpu().numpy().T)

    def zeros(self, rows, cols):
        return torch.zeros((cols, rows), dtype=torch.float64, device=self.device)

    def _p(self, t):
        import ctypes
        return ctypes.c_void_p(t.data_ptr())

    def _stream(self):
        import ctypes
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    # -- kernels
    def gemm(self, A, B, C, alpha=1.0, beta=0.0, ta=False, tb=False):
        """C = alpha op(A) op(B) + beta C on column-major views (tensors (cols, rows))."""
        lda, ldb, ldc = A.stride(0), B.stride(0), C.stride(0)
        m = A.shape[0] if ta else A.shape[1]
        k = A.shape[1] if ta else A.shape[0]
        n = B.shape[1] if tb else B.shape[0]
        ws = getattr(self, "_ws", None)
        if ws is None:
            ws = self._ws = torch.empty(64 << 20, dtype=torch.uint8, device=self.device)
        rc = self.L.pevd_dgemm(int(ta), int(tb), m, n, k, alpha, self._p(A), lda, self._p(B), ldb,
                               beta, self._p(C), ldc, self._p(ws), ws.numel(), self._stream())
        self._lib.check(rc, "dgemm")

    def panel_qr(self, P):
        """Householder QR of the column-major panel P (pw, m): returns (R, Y, T) as tensors."""
        pw, m = P.shape
        R = torch.empty((pw, pw), dtype=torch.float64, device=self.device)
        Y = torch.empty((pw, m), dtype=torch.float64, device=self.device)
        T = torch.empty((pw, pw), dtype=torch.float64, device=self.device)
        ws = torch.empty(self.L.pevd_panel_qr_workspace_bytes(), dtype=torch.uint8, device=self.device)
        rc = self.L.pevd_panel_qr(m, pw, self._p(P), P.stride(0), self._p(R), self._p(Y), m, None, m,
                                  self._p(T), self._p(ws), self._stream())
        self._lib.check(rc, "panel_qr")
        return R, Y, T

    def bc(self, bands):
        """bands (b+1, n) device tensor -> (d, e) host arrays, (tau, V) device tensors."""
        b, n = bands.shape[0] - 1, bands.shape[1]
        bands = bands.contiguous()
        d = torch.empty(n, dtype=torch.float64, device=self.device)
        e = torch.empty(max(n, 2), dtype=torch.float64, device=self.device)
        nref = max(self.L.pevd_bc_num_reflectors(n, b), 1)
        vld = ((b + 7) // 8) * 8
        tau = torch.zeros(nref, dtype=torch.float64, device=self.device)
        V = torch.zeros(nref * vld, dtype=torch.float64, device=self.device)
        ws = torch.empty(self.L.pevd_bc_workspace_bytes(n, b), dtype=torch.uint8, device=self.device)
        rc = self.L.pevd_bc(n, b, self._p(bands), self._p(d), self._p(e), self._p(tau), self._p(V),
                            vld, self._p(ws), self._stream())
        self._lib.check(rc, "bc")
        return d, e[: n - 1], tau, (V, vld)

    def stedc(self, d, e, cols=None):
        """Device divide and conquer on (d, e) device tensors -> (lam host, Q_d device); with
        cols = (c0, c1) only those eigenvector columns are formed (the rest stays zero)."""
        n = d.shape[0]
        dd = d.clone()
        ee = e.clone() if n > 1 else torch.zeros(1, dtype=torch.float64, device=self.device)
        Q = torch.empty((n, n), dtype=torch.float64, device=self.device)
        ws = torch.empty(self.L.pevd_stedc_workspace_bytes(n), dtype=torch.uint8, device=self.device)
        if cols is None:
            rc = self.L.pevd_stedc(n, self._p(dd), self._p(ee), self._p(Q), n, self._p(ws),
                                   self._stream())
        else:
            rc = self.L.pevd_stedc_cols(n, self._p(dd), self._p(ee), self._p(Q), n, int(cols[0]),
                                        int(cols[1]), self._p(ws), self._stream())
        if rc == self._lib.PEVD_ERR_CONVERGE:
            raise RuntimeError(self.L.pevd_last_error().decode())
        self._lib.check(rc, "stedc")
        return dd.cpu().numpy(), Q

    def bc_back_left(self, n, b, tau, Vpack, X):
        """X (column-major n x cols device tensor) <- Q_b X in place (conventional BC-Back)."""
        V, vld = Vpack
        cols = X.shape[0]
        ws = torch.empty(self.L.pevd_bc_back_workspace_bytes(n, cols), dtype=torch.uint8,
                         device=self.device)
        rc = self.L.pevd_bc_back_left(n, b, self._p(tau), self._p(V), vld, self._p(X),
                                      X.stride(0), cols, self._p(ws), self._stream())
        self._lib.check(rc, "bc_back_left")
        return X

    def bc_back_right(self, n, b, tau, Vpack, X):
        """X (column-major rows x n device tensor) <- X Q_b in place."""
        V, vld = Vpack
        rows = X.shape[1]
        ws = torch.empty(self.L.pevd_bc_back_workspace_bytes(n, rows), dtype=torch.uint8,
                         device=self.device)
        rc = self.L.pevd_bc_back_right(n, b, self._p(tau), self._p(V), vld, self._p(X),
                                       X.stride(0), rows, self._p(ws), self._stream())
        self._lib.check(rc, "bc_back_right")
        return X


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


def run_distributed(a, cfg, ops=None, group=None, n=None, gather_q=True):
    """Blockwise multi-process EVD.

    `a` is either the full matrix (every rank passes the same one; validated like the reference)
    or, for device-resident runs, a callable ``a(c0, c1)`` returning this rank's column block as
    a column-major device tensor of shape (c1 - c0, n) (then `n` must be given).  Every rank gets
    the eigenvalues; with gather_q the full Q (C order) too, else only its row block.

    Returns (EigenResult, events, ledger, info dict)."""
    if ops is None:
        ops = CudaOps()
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

    def factor(c0, pw, t0):
        """Gather the panel at its owner (pieces of straddling panels, C2), factor it there,
        return the R pieces (C3) and broadcast the factor (C4).  Returns (Y, T)."""
        m = n - t0
        owner = owner_of(c0)
        if rank == owner:
            P = ops.zeros(m, pw)
            hi = min(c0 + pw, c1w)
            P[: hi - c0] = blk[c0 - c0w: hi - c0w, t0:]
        for x in range(G):
            xlo, xhi = max(c0, ranges[x][0]), min(c0 + pw, ranges[x][1])
            if x == owner or xlo >= xhi:
                continue
            ledger.record(x, owner, "SBR-panel", (xhi - xlo) * m)
            if rank == x:
                _send(blk[xlo - c0w: xhi - c0w, t0:].contiguous(), owner, group)
            elif rank == owner:
                piece = torch.empty((xhi - xlo, m), dtype=torch.float64, device=blk.device)
                _recv(piece, x, group)
                P[xlo - c0: xhi - c0] = piece
        if rank == owner:
            R, Y, T = ops.panel_qr(P)
            Rfull = torch.zeros((pw, m), dtype=torch.float64, device=blk.device)
            Rfull[:, :pw] = R  # panel rows t0.. become [R; 0]
            hi = min(c0 + pw, c1w)
            blk[c0 - c0w: hi - c0w, t0:] = Rfull[: hi - c0]
        else:
            Y = torch.empty((pw, m), dtype=torch.float64, device=blk.device)
            T = torch.empty((pw, pw), dtype=torch.float64, device=blk.device)
        for x in range(G):
            xlo, xhi = max(c0, ranges[x][0]), min(c0 + pw, ranges[x][1])
            if x == owner or xlo >= xhi:
                continue
            ledger.record(owner, x, "SBR-panel", (xhi - xlo) * m)
            if rank == owner:
                _send(Rfull[xlo - c0: xhi - c0].contiguous(), x, group)
            elif rank == x:
                piece = torch.empty((xhi - xlo, m), dtype=torch.float64, device=blk.device)
                _recv(piece, owner, group)
                blk[xlo - c0w: xhi - c0w, t0:] = piece
        _bcast(Y, owner, group)
        _bcast(T, owner, group)
        ledger.record(owner, BROADCAST, "SBR", 2 * m * pw)  # the reference ships (W, Y)
        return Y, T

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
            Y, T = factor(c0, pw, t0)
            W = ops.zeros(n - t0, pw)
            ops.gemm(Y, T, W)  # W = Y T
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
            Y, T = factor(ci, b, ti)
            W = ops.zeros(n - ti, b)
            ops.gemm(Y, T, W)
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
    trace.add(rank, "SBR", rank, t_sbr0, now())

    # ---- band: our columns' diagonals, all-gathered (replaces C6/C7) ----
    width = c1w - c0w
    own_bands = torch.zeros((width, b + 1), dtype=torch.float64, device=blk.device)
    for d in range(b + 1):
        nv = min(width, n - d - c0w)
        if nv > 0:
            j = torch.arange(nv, device=blk.device)
            own_bands[:nv, d] = blk[j, c0w + d + j]
    counts = [hi - lo for lo, hi in ranges]
    bands_rows = _allgather_uneven(own_bands, counts, group, (b + 1,))  # (n, b+1)
    for w in range(G):
        ledger.record(w, HOST, "BandStage", (b + 1) * counts[w])
    bands = bands_rows.t().contiguous()                                # (b+1, n)
    # ---- BC on every rank (deterministic wavefront chase) ----
    t_bc = now()
    d, e, tau, V = ops.bc(bands)
    trace.add(rank, "BC", rank, t_bc, now())
    for w in range(G - 1):
        ledger.record(w, w + 1, "BC", 2 * b * b)  # the overlap-block hand-off of the relay
    # ---- solver ----
    t_s = now()
    # (conventional order: each rank forms only its own columns of Q_d)
    if cfg.order == "conventional" and cfg.want_vectors:
        lam, Qd = ops.stedc(d, e, cols=(c0w, c1w))
    else:
        lam, Qd = ops.stedc(d, e)  # lam on the host, Q_d column-major (device for CudaOps)
    trace.add(HOST, "Solver", 0, t_s, now())
    if not cfg.want_vectors:
        return EigenResult(lam=lam), trace.events(), ledger, {}
    if cfg.order == "conventional":
        # ---- conventional order by columns: Q[:, ours] = Q_s Q_b Q_d[:, ours].  Every rank
        #      already holds Q_d, the bulge reflectors and the SBR panels, so the column blocks
        #      are independent: no Q_d / U broadcasts, no final GEMM (pipeline.py:367-387) ----
        t_bb = now()
        X = Qd[c0w:c1w].clone()                       # column-major n x (c1w - c0w)
        X = ops.bc_back_left(n, b, tau, V, X)         # Q_b X
        trace.add(rank, "BC-Back", rank, t_bb, now())
        t_sb = now()
        groups = [panels[g0:g0 + SBR_BACK_AGG] for g0 in range(0, len(panels), SBR_BACK_AGG)]
        for grp in reversed(groups):                  # Q_s X = H_0 (H_1 (... X))
            t0, Yg, Tg = _aggregate(ops, grp, n)
            K = Tg.shape[0]
            X2 = X[:, t0:]                            # rows t0.. of our columns
            P1 = ops.zeros(K, c1w - c0w)
            ops.gemm(Yg, X2, P1, ta=True)             # Y^T X
            P2 = ops.zeros(K, c1w - c0w)
            ops.gemm(Tg, P1, P2)                      # T (Y^T X)
            ops.gemm(Yg, P2, X2, alpha=-1.0, beta=1.0)  # X -= Y T Y^T X
        trace.add(rank, "SBR-Back", rank, t_sb, now())
        if not gather_q:
            return (EigenResult(lam=lam), trace.events(), ledger,
                    {"cols": (c0w, c1w), "q_cols": X})
        counts = [hi - lo for lo, hi in ranges]
        Qc = _allgather_uneven(X, counts, group, (n,))   # (n cols, n rows): column-major Q
        for w in range(G):
            ledger.record(w, HOST, "Result", counts[w] * n)
        return (EigenResult(lam=lam, Q=np.asfortranarray(Qc.cpu().numpy().T),
                            vectors_computed=True),
                trace.events(), ledger, {"cols": (c0w, c1w)})
    # ---- back transformation of our rows ----
    sizes = back_plan_sizes(n, G, cfg.back_skew)
    bounds = np.cumsum([0] + sizes)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
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
    trace.add(rank, "SBR-Back", rank, t_sb, now())
    t_bb = now()
    Msb = ops.bc_back_right(n, b, tau, V, Mt)   # rows of Q_s Q_b (in place)
    trace.add(rank, "BC-Back", rank, t_bb, now())
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
