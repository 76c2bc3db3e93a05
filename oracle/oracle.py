"""CPU oracle for the pipelined two-stage FP64 EVD -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference package `pipeevd` (paths below are
relative to /root/reference/pkg/src/pipeevd) plus the C restatement of its
three scalar numba kernels (oracle/pevd_oracle.c -> oracle/liboracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
as the timed CPU baseline.  The product package never imports it.

Parity is PINNED: tests/test_oracle.py checks every function here against
golden vectors produced by the real reference (tests/golden/make_golden.py,
run in the build container where /root/reference exists) and against the
reference's own known-answer tests.
"""
from __future__ import annotations

import ctypes
import os
import math

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

EPS = float(np.finfo(np.float64).eps)
MAX_ITER_PER_N = 30          # tridiag.py:23
DEFAULT_GROUP_SIZE = 4       # backtrans.py:23

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


def lib():
    """Load (building if needed) the C restatement of the numba kernels."""
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            import subprocess
            subprocess.run(["make", "-C", _HERE, "-s"], check=True)
        L = ctypes.CDLL(path)
        L.orc_chase.restype = ctypes.c_int64
        L.orc_chase.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                _i64p, _i64p, _i64p, _i64p, _f64p, _f64p,
                                ctypes.c_int64, _i64p]
        L.orc_steqr.restype = ctypes.c_int64
        L.orc_steqr.argtypes = [_f64p, _f64p, ctypes.c_int64, _f64p, ctypes.c_int64,
                                ctypes.c_int64, _i64p, _i64p]
        L.orc_rank1_seq.restype = ctypes.c_int64
        L.orc_rank1_seq.argtypes = [_f64p, ctypes.c_int64, _i64p, ctypes.c_int64,
                                    _i64p, _i64p, _f64p, _f64p, ctypes.c_int64, _f64p]
        _LIB = L
    return _LIB


def _p(a, t=_f64p):
    return a.ctypes.data_as(t)


def pad8(k: int) -> int:
    """bulge.py:29-30"""
    return ((k + 7) // 8) * 8


# --------------------------------------------------------------------------
# core.py


def house_vector(x):
    """core.py:238-255: (v, tau, alpha) with v[0]=1, alpha=-sign(x0)||x||, sign(0)=+."""
    x = np.asarray(x, dtype=np.float64)
    v = np.zeros(len(x))
    v[0] = 1.0
    tail = float(np.linalg.norm(x[1:]))
    if tail == 0.0:
        return v, 0.0, float(x[0])
    alpha = (-1.0 if x[0] >= 0.0 else 1.0) * float(np.hypot(x[0], tail))
    v[1:] = x[1:] / (x[0] - alpha)
    tau = 2.0 / (1.0 + float(np.dot(v[1:], v[1:])))
    return v, tau, alpha


def band_from_dense(a, b):
    """core.py:138-146: bands[d, j] = A[j+d, j]."""
    n = a.shape[0]
    bands = np.zeros((b + 1, n))
    for d in range(b + 1):
        bands[d, : n - d] = np.diagonal(a, -d)
    return bands


def band_to_dense(bands):
    """core.py:148-155"""
    b = bands.shape[0] - 1
    n = bands.shape[1]
    a = np.zeros((n, n))
    for d in range(b + 1):
        idx = np.arange(n - d)
        a[idx + d, idx] = bands[d, : n - d]
        a[idx, idx + d] = bands[d, : n - d]
    return a


# --------------------------------------------------------------------------
# sbr.py


def round_schedule(n, b):
    """sbr.py:54-66: (col_start, panel_width, trailing_start) per round."""
    out, c0 = [], 0
    while c0 < n - b:
        out.append((c0, min(b, n - b - c0), c0 + b))
        c0 += b
    return out


def panel_qr(panel, inner_block=8):
    """sbr.py:69-116: blocked Householder QR; panel <- R, returns (W, Y)."""
    m, k = panel.shape
    W = np.zeros((m, k), order="F")
    Y = np.zeros((m, k), order="F")
    for j0 in range(0, k, inner_block):
        j1 = min(j0 + inner_block, k)
        wb = np.zeros((m, j1 - j0), order="F")
        for j in range(j0, j1):
            v, tau, alpha = house_vector(panel[j:, j])
            Y[j:, j] = v
            panel[j, j] = alpha
            panel[j + 1:, j] = 0.0
            rest = panel[j:, j + 1:j1]
            if tau != 0.0 and rest.shape[1]:
                rest -= np.outer(tau * v, v @ rest)
            vf = Y[:, j]
            W[:, j] = tau * (vf - W[:, :j] @ (Y[:, :j].T @ vf)) if j > 0 else tau * vf
            wb[:, j - j0] = (tau * (vf - wb[:, :j - j0] @ (Y[:, j0:j].T @ vf))
                             if j > j0 else tau * vf)
        rest = panel[:, j1:]
        if rest.shape[1]:
            rest -= Y[:, j0:j1] @ (wb.T @ rest)
    return W, Y


def form_z(a2, W, Y):
    """sbr.py:119-130: Z = A W - Y (W^T A W)/2."""
    aw = a2 @ W
    return aw - 0.5 * (Y @ (W.T @ aw))


def trailing_update(a2, Y, Z):
    """sbr.py:133-152 / core.py:282-306: A2 -= Y Z^T + Z Y^T, lower triangle
    computed, mirrored bit-exactly onto the upper one."""
    upd = Y @ Z.T
    a2 -= upd + upd.T
    il = np.tril_indices(a2.shape[0], -1)
    a2.T[il] = a2[il]


def sbr_reduce(a, b, inner_block=8):
    """sbr.py:155-188: dense -> band; returns (bands (b+1, n), [(c0, W, Y)])."""
    n = a.shape[0]
    work = np.array(a, dtype=np.float64, order="F")
    panels = []
    for c0, pw, t0 in round_schedule(n, b):
        panel = work[t0:, c0:c0 + pw]
        W, Y = panel_qr(panel, inner_block)
        work[c0:c0 + pw, t0:] = panel.T
        if pw < b:
            cp = work[t0:, c0 + pw:t0]
            if cp.shape[1]:
                cp -= Y @ (W.T @ cp)
                work[c0 + pw:t0, t0:] = cp.T
        tr = work[t0:, t0:]
        Z = form_z(tr, W, Y)
        trailing_update(tr, Y, Z)
        panels.append((c0, W, Y))
    return band_from_dense(work, b), panels


# --------------------------------------------------------------------------
# bulge.py


def step_capacity(n, b, i0=0, i1=None):
    """bulge.py:255-259"""
    i1 = n if i1 is None else i1
    return sum((n - 3 - i) // b + 1 for i in range(i0, min(i1, n - 2)))


def bc_reduce(bands):
    """bulge.py:299-309: band -> (d, e, reflectors) with reflectors a dict of
    arrays i, j, row0, len, tau, v in canonical (j outer, i inner) order."""
    b = bands.shape[0] - 1
    n = bands.shape[1]
    stride = pad8(max(b, 1))
    if b <= 1:
        d = bands[0].copy()
        e = bands[1, : n - 1].copy() if b == 1 else np.zeros(max(n - 1, 0))
        z = np.zeros(0, dtype=np.int64)
        return d, e, dict(i=z, j=z, row0=z, len=z, tau=np.zeros(0), v=np.zeros((0, stride)))
    s = np.ascontiguousarray(band_to_dense(bands))
    cap = max(step_capacity(n, b), 1)
    ia = np.zeros(cap, np.int64); ja = np.zeros(cap, np.int64)
    ra = np.zeros(cap, np.int64); la = np.zeros(cap, np.int64)
    ta = np.zeros(cap); va = np.zeros((cap, stride))
    macs = ctypes.c_int64(0)
    cnt = lib().orc_chase(_p(s), n, 0, n, b, 0, n, _p(ia, _i64p), _p(ja, _i64p),
                          _p(ra, _i64p), _p(la, _i64p), _p(ta), _p(va), stride,
                          ctypes.byref(macs))
    perm = np.lexsort((ia[:cnt], ja[:cnt]))
    refl = dict(i=ia[:cnt][perm], j=ja[:cnt][perm], row0=ra[:cnt][perm],
                len=la[:cnt][perm], tau=ta[:cnt][perm], v=va[:cnt][perm])
    return np.diag(s).copy(), np.diag(s, -1).copy(), refl


# --------------------------------------------------------------------------
# tridiag.py


def tridiag_eig(d, e, want_vectors=False):
    """tridiag.py:298-334: (lam ascending, Q with sign convention or None)."""
    n = len(d)
    dd = np.array(d, dtype=np.float64)
    ee = np.zeros(max(n, 1))
    ee[: n - 1] = e
    zt = np.eye(n) if want_vectors else np.zeros((1, 1))
    tot = ctypes.c_int64(0); rots = ctypes.c_int64(0)
    failed = lib().orc_steqr(_p(dd), _p(ee), n, _p(zt), n if want_vectors else 0,
                             MAX_ITER_PER_N * n, ctypes.byref(tot), ctypes.byref(rots))
    if failed >= 0:
        raise RuntimeError(f"tridiagonal QL/QR did not converge near index {failed}")
    perm = np.argsort(dd, kind="stable")
    lam = dd[perm].copy()
    if not want_vectors:
        return lam, None
    q = np.asfortranarray(zt[perm].T)
    for jc in range(n):
        col = q[:, jc]
        if col[int(np.argmax(np.abs(col)))] < 0.0:
            np.negative(col, out=col)
    return lam, q


# --------------------------------------------------------------------------
# backtrans.py


def sbr_back_rows(n, panels, rows):
    """backtrans.py:149-192: rows [lo, hi) of Q_s by forward panel application."""
    lo, hi = rows
    m = np.zeros((hi - lo, n))
    m[np.arange(hi - lo), np.arange(lo, hi)] = 1.0
    for c0, W, Y in panels:
        t0 = n - W.shape[0]
        blk = m[:, t0:]
        blk -= (blk @ W) @ Y.T
    return m


def sbr_back_accumulate(n, panels, cols):
    """backtrans.py:128-146: columns [lo, hi) of Q_s."""
    lo, hi = cols
    q = np.zeros((n, hi - lo), order="F")
    q[np.arange(lo, hi), np.arange(hi - lo)] = 1.0
    for c0, W, Y in reversed(panels):
        t0 = n - W.shape[0]
        blk = q[t0:, :]
        blk -= W @ (Y.T @ blk)
    return q


def application_order(refl, direction="reordered", grouped=True,
                      group_size=DEFAULT_GROUP_SIZE):
    """backtrans.py:214-236"""
    i, j = refl["i"], refl["j"]
    if len(i) == 0:
        return np.zeros(0, dtype=np.int64)
    k = i // group_size
    if direction == "reordered":
        return np.lexsort((i, -j, k)) if grouped else np.lexsort((j, i))
    if direction == "conventional":
        return np.lexsort((-i, j, -k)) if grouped else np.lexsort((j, i))[::-1].copy()
    raise ValueError(direction)


def bc_back_apply(refl, x, direction="reordered", grouped=True,
                  group_size=DEFAULT_GROUP_SIZE):
    """backtrans.py:277-310: Q_b^T X (reordered) or Q_b X (conventional)."""
    q = np.array(x, dtype=np.float64, order="C")
    if len(refl["tau"]) == 0:
        return q
    order = np.ascontiguousarray(application_order(refl, direction, grouped, group_size),
                                 dtype=np.int64)
    dots = np.empty(q.shape[1])
    v = np.ascontiguousarray(refl["v"])
    lib().orc_rank1_seq(_p(q), q.shape[1], _p(order, _i64p), len(order),
                        _p(np.ascontiguousarray(refl["row0"]), _i64p),
                        _p(np.ascontiguousarray(refl["len"]), _i64p),
                        _p(np.ascontiguousarray(refl["tau"])), _p(v), v.shape[1], _p(dots))
    return q


# --------------------------------------------------------------------------
# the whole single-worker EVD (pipeline.py:511 semantics with workers=1)


def evd(a, b=32, want_vectors=True, order="pipelined"):
    """Single-worker restatement of pipeline.run: returns (lam, Q or None).

    pipelined/sequential: Q = (Q_s Q_b) Q_d via the reordered transform
    (pipeline.py:398-418); conventional: Q = Q_s (Q_b Q_d) (pipeline.py:367-387).
    """
    a = np.asarray(a, dtype=np.float64)
    n = a.shape[0]
    if n == 1:
        return a[0].copy().reshape(1), (np.ones((1, 1)) if want_vectors else None)
    b = min(b, n - 1)
    bands, panels = sbr_reduce(a, b)
    d, e, refl = bc_reduce(bands)
    lam, qd = tridiag_eig(d, e, want_vectors)
    if not want_vectors:
        return lam, None
    if order == "conventional":
        zb = bc_back_apply(refl, qd, direction="conventional")
        for c0, W, Y in reversed(panels):
            mp = W.shape[0]
            blk = zb[n - mp:, :]
            blk -= W @ (Y.T @ blk)
        return lam, np.asfortranarray(zb)
    m = sbr_back_rows(n, panels, (0, n))
    ub = bc_back_apply(refl, m.T)
    return lam, np.ascontiguousarray(ub.T @ qd)


def backward_error(a, q, lam):
    """verify.py:24-34: ||A - Q diag(lam) Q^T||_F / (n ||A||_F)."""
    n = a.shape[0]
    s = float(np.linalg.norm(a))
    r = float(np.linalg.norm(a - (q * lam) @ q.T))
    return 0.0 if s == 0.0 and r == 0.0 else r / (n * s)


def orthogonality(q):
    """verify.py:37-41: ||I - Q Q^T||_F / n."""
    n = q.shape[0]
    return float(np.linalg.norm(np.eye(n) - q @ q.T)) / n
