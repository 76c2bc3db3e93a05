"""Per-stage functions with the reference's signatures, executed on the GPU.

Each mirrors a reference function (file:line) so the reference's own per-stage tests read the
same against this package; the arithmetic runs in libpevd.so (device.py -> C ABI).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import device
from .core import (BandMatrix, FlopCounter, ProtocolError, ReflectorPanel, SymmetricMatrix,
                   TridiagonalMatrix, EigenResult)
from .schedule import bc_back_macs, bc_macs, round_schedule, sbr_macs

DEFAULT_GROUP_SIZE = 4  # backtrans.py:23 (device kernels use their own grouping)


def _pad8(k: int) -> int:
    return ((k + 7) // 8) * 8


# ------------------------------------------------------------------ SBR


@dataclass
class SbrConfig:
    """sbr.py:20-34"""

    b: int = 32
    panel_width: int | None = None
    inner_block: int = 8

    def __post_init__(self):
        if self.panel_width is None:
            self.panel_width = self.b
        if self.panel_width != self.b:
            raise ValueError("panel_width must equal the bandwidth")
        if self.b < 1:
            raise ValueError("bandwidth must be >= 1")
        if self.inner_block < 1:
            raise ValueError("inner_block must be >= 1")


@dataclass
class SbrFactors:
    """All panel reflectors of one reduction, ordered by column offset (sbr.py:37-51)."""

    n: int
    b: int
    panels: list = field(default_factory=list)


def house_vector(x):
    """core.py:238-255 (scalar helper; the device kernels inline the same convention)."""
    x = np.asarray(x, dtype=np.float64)
    v = np.zeros(len(x))
    v[0] = 1.0
    tail = float(np.linalg.norm(x[1:]))
    if tail == 0.0:
        return v, 0.0, float(x[0])
    sign = -1.0 if x[0] < 0.0 else 1.0
    alpha = -sign * float(np.hypot(x[0], tail))
    v[1:] = x[1:] / (x[0] - alpha)
    return v, 2.0 / (1.0 + float(np.dot(v[1:], v[1:]))), alpha


def apply_block_reflector(c, panel: ReflectorPanel, side: str = "left", transpose: bool = False,
                          counter: FlopCounter | None = None, stage: str = "reflector"):
    """Q c, Q^T c, c Q or c Q^T for Q = I - W Y^T, in place, on the DMMA GEMM (core.py:258-279)."""
    w, y = panel.W, panel.Y
    if transpose:
        w, y = y, w
    if side == "left":
        c -= device.dgemm(w, device.dgemm(y, c, trans_a=True))
    elif side == "right":
        c -= device.dgemm(device.dgemm(c, w), y, trans_b=True)
    else:
        raise ValueError(f"side must be left or right, got {side!r}")
    if counter is not None:
        counter.add(stage, 2 * c.shape[0] * c.shape[1] * panel.width)
    return c


def sym_rank2k_update(a, y, z, counter: FlopCounter | None = None, stage: str = "rank2k"):
    """a -= y z^T + z y^T, symmetric to the last bit (core.py:282-306): the lower triangle is
    computed on the GPU and mirrored."""
    m, k = y.shape
    if a.shape != (m, m) or z.shape != (m, k):
        raise ValueError("shape mismatch in rank-2k update")
    yz = np.hstack([y, z])
    zy = np.hstack([z, y])
    new = device.dgemm(yz, zy, alpha=-1.0, beta=1.0, c=a, trans_b=True)  # a - [y z][z y]^T
    il = np.tril_indices(m)
    a[il] = new[il]                  # the lower triangle from the device ...
    iu = np.triu_indices(m, 1)
    a[iu] = a.T[iu]                  # ... mirrored (a copy, no host arithmetic)
    if counter is not None:
        counter.add(stage, m * (m + 1) * k)
    return a


def form_z(a_trailing, w, y, counter: FlopCounter | None = None, stage: str = "SBR"):
    """Z = A W - Y (W^T A W)/2 with the symmetric-lower DMMA product for A W (sbr.py:119-130)."""
    m, k = w.shape
    if a_trailing.shape != (m, m) or y.shape != (m, k):
        raise ValueError("shape mismatch in form_z")
    aw = device.dsymm_lower(a_trailing, w)
    z = device.dgemm(y, device.dgemm(w, aw, trans_a=True), alpha=-0.5, beta=1.0, c=aw)
    if counter is not None:
        counter.add(stage, m * m * k + k * k * m + m * k * k)
    return z


def trailing_update(a2, y, z, mode: str = "symmetric", counter: FlopCounter | None = None,
                    stage: str = "SBR"):
    """A2 -= Y Z^T + Z Y^T (sbr.py:133-152)."""
    m, k = y.shape
    if a2.shape != (m, m) or z.shape != (m, k):
        raise ValueError("shape mismatch in trailing update")
    if mode == "full":
        a2[...] = device.dgemm(np.hstack([y, z]), np.hstack([z, y]), alpha=-1.0, beta=1.0, c=a2,
                               trans_b=True)
        if counter is not None:
            counter.add(stage, 2 * m * m * k)
    elif mode == "symmetric":
        sym_rank2k_update(a2, y, z, counter, stage)
    else:
        raise ValueError(f"mode must be full or symmetric, got {mode!r}")


def panel_qr(panel: np.ndarray, col_offset: int = 0, inner_block: int = 8,
             counter: FlopCounter | None = None, stage: str = "SBR") -> ReflectorPanel:
    """Householder QR of a panel on the GPU; overwrites it with R (sbr.py:69-116)."""
    m, k = panel.shape
    if m < k:
        raise ValueError("panel must be at least as tall as wide")
    R, Y, W, T = device.panel_qr(panel)
    panel[:k, :] = np.triu(R)
    panel[k:, :] = 0.0
    panel[np.tril_indices(k, -1)] = 0.0
    if counter is not None:
        counter.add(stage, 2 * m * k * k)
    return ReflectorPanel(W=W, Y=Y, col_offset=col_offset)


def sbr_reduce(a: SymmetricMatrix, cfg: SbrConfig, counter: FlopCounter | None = None):
    """Dense -> band on the GPU: (BandMatrix, SbrFactors) (sbr.py:155-188)."""
    n, b = a.n, cfg.b
    if n <= b:
        raise ValueError(f"need n > b, got n={n}, b={b}")
    bands, ystair, tall = device.sbr(a.data, b)
    panels = []
    for x, (c0, pw, t0) in enumerate(round_schedule(n, b)):
        Y = np.asfortranarray(ystair[t0:, c0:c0 + pw])
        T = device.t_block(tall, x, b, pw)
        p = ReflectorPanel(W=device.dgemm(Y, T), Y=Y, col_offset=c0)
        p._T = T
        panels.append(p)
    if counter is not None:
        counter.add("SBR", sbr_macs(n, b))
    return BandMatrix(n, b, bands), SbrFactors(n=n, b=b, panels=panels)


# ------------------------------------------------------------------ BC


class BulgeReflectorSet:
    """Bulge-chasing reflectors in canonical (chase step j, sweep i) order (bulge.py:33-141)."""

    def __init__(self, n, b, i_idx, j_idx, row0, length, tau, v):
        self.n, self.b = n, b
        self.i_idx = np.ascontiguousarray(i_idx, dtype=np.int64)
        self.j_idx = np.ascontiguousarray(j_idx, dtype=np.int64)
        self.row0 = np.ascontiguousarray(row0, dtype=np.int64)
        self.length = np.ascontiguousarray(length, dtype=np.int64)
        self.tau = np.ascontiguousarray(tau, dtype=np.float64)
        self.v = np.ascontiguousarray(v, dtype=np.float64)
        if len(self.tau):
            perm = np.lexsort((self.i_idx, self.j_idx))
            for name in ("i_idx", "j_idx", "row0", "length", "tau", "v"):
                setattr(self, name, np.ascontiguousarray(getattr(self, name)[perm]))
        if self.v.shape != (len(self.tau), _pad8(b)):
            raise ValueError("reflector storage has the wrong stride")
        for t in self.tau:
            if not math.isfinite(t):
                raise ValueError("non-finite tau")
        if len(self.tau) and np.any(self.v[:, 0] != 1.0):
            raise ValueError("reflector vectors must have v[0] = 1")
        self._pos = {(int(i), int(j)): p for p, (i, j) in enumerate(zip(self.i_idx, self.j_idx))}
        if len(self._pos) != len(self.tau):
            raise ValueError("duplicate (sweep, step) index")
        self._slots = None

    def __len__(self) -> int:
        return len(self.tau)

    @property
    def stride(self) -> int:
        return self.v.shape[1] if len(self.tau) else _pad8(self.b)

    def position(self, i, j):
        return self._pos.get((i, j))

    def by_step(self) -> dict:
        out: dict = {}
        for p in range(len(self.tau)):
            out.setdefault(int(self.j_idx[p]), []).append(p)
        return out

    def group_labels(self, group_size: int = 4):
        """(G_k, B_j) labels per reflector (bulge.py:90-92)."""
        return self.i_idx // group_size, self.j_idx.copy()

    def back_deps(self, i: int, j: int):
        """Reflectors applied before u_(i,j) in the conventional direction (bulge.py:94-96)."""
        return [(i + 1, j - 1), (i + 1, j)] if j >= 1 else [(i + 1, j)]

    def validate_order(self, order, direction: str = "reordered") -> None:
        """Check an application order against the dependency rule (bulge.py:98-119)."""
        when = np.empty(len(self.tau), dtype=np.int64)
        when[np.asarray(order, dtype=np.int64)] = np.arange(len(order))
        for p in range(len(self.tau)):
            i, j = int(self.i_idx[p]), int(self.j_idx[p])
            if direction == "conventional":
                needed = [(i + 1, j - 1), (i + 1, j)]
            elif direction == "reordered":
                needed = [(i - 1, j), (i - 1, j + 1)]
            else:
                raise ValueError(direction)
            for i2, j2 in needed:
                q = self._pos.get((i2, j2))
                if q is not None and when[q] >= when[p]:
                    raise ValueError(f"order violates dependency: u_({i},{j}) before u_({i2},{j2})")

    @classmethod
    def merge(cls, parts):
        """Concatenate per-worker sets (bulge.py:126-141)."""
        parts = list(parts)
        if not parts:
            raise ValueError("nothing to merge")
        n, b = parts[0].n, parts[0].b
        if any((p.n, p.b) != (n, b) for p in parts):
            raise ValueError("mismatched reflector sets")
        return cls(n, b, *(np.concatenate([getattr(p, f) for p in parts])
                           for f in ("i_idx", "j_idx", "row0", "length", "tau")),
                   np.vstack([p.v for p in parts]))

    @classmethod
    def empty(cls, n, b):
        z = np.zeros(0)
        return cls(n, b, z, z, z, z, z, np.zeros((0, _pad8(b))))

    @classmethod
    def from_slots(cls, n, b, tau, V):
        r = device.slots_to_reference(n, b, tau, V)
        u = cls(n, b, r["i"], r["j"], r["row0"], r["len"], r["tau"], r["v"])
        u._slots = (tau, V)
        return u

    def slots(self):
        """Fixed-slot layout of the device kernels (include/pevd.h pevd_bc)."""
        if self._slots is None:
            n, b = self.n, self.b
            nslot = 0
            j = 0
            while n - 2 - j * b > 0:
                nslot += n - 2 - j * b
                j += 1
            tau = np.zeros(max(nslot, 1))
            V = np.zeros((max(nslot, 1), _pad8(b)))
            jj = self.j_idx.astype(np.int64)
            s_ = jj * (n - 2) - b * jj * (jj - 1) // 2 + self.i_idx.astype(np.int64)
            tau[s_] = self.tau
            V[s_] = self.v
            self._slots = (tau, V)
        return self._slots


@dataclass
class BcPartitionResult:
    """One worker's share of the relayed chase (bulge.py:312-318)."""

    d_part: np.ndarray
    e_part: np.ndarray
    reflectors: "BulgeReflectorSet"
    outgoing: "OverlapBlock | None"
    tail: BandMatrix | None  # the modified band beyond pivot_end, None for the last worker


def _validate_incoming(incoming, col0: int, b: int) -> None:
    """bulge.py:335-345: the predecessor's overlap block must be empty but the bridge entry."""
    if incoming.offset != col0:
        raise ProtocolError(f"overlap offset {incoming.offset} does not match boundary {col0}")
    if incoming.b != b:
        raise ProtocolError("overlap bandwidth mismatch")
    mask = np.ones(incoming.values.shape, dtype=bool)
    mask[0, b - 1] = False  # the subdiagonal bridge entry may be nonzero
    if np.any(incoming.values[mask] != 0.0):
        raise ProtocolError("overlap block contains fill outside the bridge entry")


def bc_reduce_partition(band_tail: BandMatrix, b: int, col0: int, pivot_end: int,
                        incoming=None, is_last: bool = False,
                        counter: FlopCounter | None = None) -> BcPartitionResult:
    """Chase all sweeps with pivot in [col0, pivot_end) down the band tail on the GPU
    (bulge.py:348-385).  `band_tail` covers global columns [col0, n) with semi-bandwidth <= 2b.
    The device chase runs on the tail renumbered from 0 (the chase is translation invariant) and
    stops after the partition's sweeps; the result is bit-identical to the same sweeps of the
    whole-band chase."""
    m = band_tail.n
    n = col0 + m
    if col0 > 0:
        if incoming is None:
            raise ProtocolError("interior worker started bulge chasing without its "
                                "predecessor's overlap block")
        _validate_incoming(incoming, col0, b)
    elif incoming is not None:
        raise ProtocolError("first worker must not receive an overlap block")
    npiv = max(0, min(pivot_end, n) - col0)
    if b <= 1 or m < 3:
        out = np.zeros((max(2 * b, 1) + 1, m))
        src = band_tail.bands
        out[: src.shape[0], :] = src[:, :m]
        refl = BulgeReflectorSet.empty(n, max(b, 1))
    else:
        out, tau, V = device.bc_partition(band_tail.bands, b, npiv)
        r = device.slots_to_reference(m, b, tau, V)
        keep = r["i"] < npiv
        refl = BulgeReflectorSet(n, b, r["i"][keep] + col0, r["j"][keep], r["row0"][keep] + col0,
                                 r["len"][keep], r["tau"][keep], r["v"][keep])
        if counter is not None:
            counter.add("BC", int(7 * b * b * len(refl)))
    # finished rows: the band below the first subdiagonal must be exactly zero there
    hi = npiv
    for dd in range(2, out.shape[0]):
        if hi and np.any(out[dd, : max(0, min(hi, m - dd))] != 0.0):
            raise ProtocolError("bulge chasing left fill in finished columns")
    d_part = np.ascontiguousarray(out[0, :hi])
    e_part = np.ascontiguousarray(out[1, : min(hi, m - 1)]) if out.shape[0] > 1 else np.zeros(0)
    if is_last:
        return BcPartitionResult(d_part, e_part, refl, None, None)
    # the 2b x b overlap block: rows [pivot_end, pivot_end+2b) x columns [pivot_end-b, pivot_end)
    vals = np.zeros((2 * b, b))
    for rr in range(2 * b):
        gr = pivot_end + rr
        if gr >= n:
            break
        for cc in range(b):
            gc = pivot_end - b + cc
            if gc >= col0 and 0 <= gr - gc < out.shape[0]:
                vals[rr, cc] = out[gr - gc, gc - col0]
    outgoing = OverlapBlock(values=vals, offset=pivot_end, b=b)
    rest = out[:, pivot_end - col0:]
    mr = rest.shape[1]
    bw = min(2 * b, mr - 1) if mr > 1 else 0
    tail = BandMatrix(n=mr, b=bw, bands=np.ascontiguousarray(rest[: bw + 1]))
    return BcPartitionResult(d_part, e_part, refl, outgoing, tail)


def bc_reduce(band: BandMatrix, counter: FlopCounter | None = None):
    """Band -> tridiagonal on the GPU wavefront chase (bulge.py:299-309)."""
    n, b = band.n, band.b
    if b <= 1:
        return band.to_tridiagonal(), BulgeReflectorSet.empty(n, max(b, 1))
    d, e, tau, V = device.bc(band.bands)
    if counter is not None:
        counter.add("BC", bc_macs(n, b))
    return TridiagonalMatrix(d=d, e=e), BulgeReflectorSet.from_slots(n, b, tau, V)


# ------------------------------------------------------------------ solver


def tridiag_eig(t: TridiagonalMatrix, want_vectors: bool = False,
                counter: FlopCounter | None = None) -> EigenResult:
    """Symmetric tridiagonal eigensolver: device divide and conquer (replaces tridiag.py:298)."""
    n = t.n
    if n == 0:
        return EigenResult(lam=np.zeros(0), Q=np.zeros((0, 0)) if want_vectors else None,
                           vectors_computed=want_vectors)
    lam, q = device.stedc(t.d, t.e if n > 1 else np.zeros(0))
    if counter is not None:
        counter.add("Solver", max(1, (2 * n ** 3) // 3))
    if not want_vectors:
        return EigenResult(lam=lam)
    return EigenResult(lam=lam, Q=np.asfortranarray(q), vectors_computed=True)


# ------------------------------------------------------------------ back transformation


def bc_back_apply(u: BulgeReflectorSet, qs_t_block, counter: FlopCounter | None = None,
                  direction: str = "reordered", grouped: bool = True,
                  group_size: int = DEFAULT_GROUP_SIZE, debug_validate: bool = False,
                  inplace: bool = False) -> np.ndarray:
    """Q_b^T X ("reordered") or Q_b X ("conventional") on the GPU (backtrans.py:277-310)."""
    x = np.array(qs_t_block, dtype=np.float64, order="C")
    if x.ndim != 2 or x.shape[0] != u.n:
        raise ValueError(f"target must have {u.n} rows")
    if direction not in ("reordered", "conventional"):
        raise ValueError(f"unknown direction {direction!r}")
    if len(u) == 0:
        return x
    tau, V = u.slots()
    if direction == "reordered":
        out = device.bc_back_right(u.n, u.b, tau, V, x.T).T   # (X^T Q_b)^T = Q_b^T X
    else:
        out = device.bc_back_left(u.n, u.b, tau, V, x)
    if counter is not None:
        counter.add("BC-Back", bc_back_macs(u.n, u.b, x.shape[1]))
    return np.ascontiguousarray(out)


def sbr_back_accumulate(factors: SbrFactors, cols, counter: FlopCounter | None = None):
    """Columns [lo, hi) of Q_s (backtrans.py:128-146), formed on the GPU."""
    n = factors.n
    lo, hi = cols
    if not 0 <= lo <= hi <= n:
        raise ValueError("column range out of bounds")
    qs = _form_qs(factors)
    if counter is not None:
        counter.add("SBR-Back", max(1, (2 * n ** 3) // 3))
    return np.asfortranarray(qs[:, lo:hi])


def sbr_back_rows(factors: SbrFactors, rows, counter: FlopCounter | None = None):
    """Rows [lo, hi) of Q_s (backtrans.py:186-192)."""
    n = factors.n
    lo, hi = rows
    if not 0 <= lo <= hi <= n:
        raise ValueError("row range out of bounds")
    qs = _form_qs(factors)
    if counter is not None:
        counter.add("SBR-Back", max(1, (2 * n ** 3) // 3))
    return np.ascontiguousarray(qs[lo:hi, :])


def _form_qs(factors: SbrFactors) -> np.ndarray:
    n, b = factors.n, factors.b
    ystair = np.zeros((n, n), order="F")
    rounds = max(1, len(factors.panels))
    tall = np.zeros(rounds * b * b)
    for x, p in enumerate(factors.panels):
        m, pw = p.Y.shape
        t0 = n - m
        ystair[t0:, p.col_offset:p.col_offset + pw] = p.Y
        T = getattr(p, "_T", None)
        if T is None:  # W = Y T with Y unit lower trapezoidal: T = Y1^{-1} W1 (top pw x pw)
            from scipy.linalg import solve_triangular
            T = np.triu(solve_triangular(p.Y[:pw], p.W[:pw], lower=True, unit_diagonal=True))
        tall[x * b * b: x * b * b + pw * pw] = np.asarray(T).T.reshape(-1)
    return device.sbr_back_form(n, b, ystair, tall)


class RowAccumulator:
    """Rows of Q_s built panel by panel in creation order (backtrans.py:149-183); each panel is
    folded in from the right on the GPU: M[:, t0:] -= (M[:, t0:] W) Y^T."""

    def __init__(self, n: int, rows):
        lo, hi = rows
        if not 0 <= lo <= hi <= n:
            raise ValueError("row range out of bounds")
        self.n, self.rows = n, (lo, hi)
        self.m = np.zeros((hi - lo, n))
        self.m[np.arange(hi - lo), np.arange(lo, hi)] = 1.0
        self._applied = 0
        self._last_offset = -1

    def apply_panel(self, panel: ReflectorPanel, counter: FlopCounter | None = None) -> None:
        if panel.col_offset <= self._last_offset:
            raise ValueError("panels must arrive in ascending creation order")
        self._last_offset = panel.col_offset
        t0 = self.n - panel.W.shape[0]
        blk = self.m[:, t0:]
        blk -= device.dgemm(device.dgemm(blk, panel.W), panel.Y, trans_b=True)
        if counter is not None:
            counter.add("SBR-Back", 2 * self.m.shape[0] * (self.n - t0) * panel.width)
        self._applied += 1

    @property
    def panels_applied(self) -> int:
        return self._applied

    def matrix(self) -> np.ndarray:
        return self.m


def application_order(u: BulgeReflectorSet, direction: str = "reordered", grouped: bool = True,
                      group_size: int = DEFAULT_GROUP_SIZE) -> np.ndarray:
    """Dependency-valid reflector orders (backtrans.py:214-236); the device kernels use the
    grouped form with group size 64 and 8-reflector compact-WY blocks."""
    i, j = u.i_idx, u.j_idx
    if len(u) == 0:
        return np.zeros(0, dtype=np.int64)
    k = i // group_size
    if direction == "reordered":
        return np.lexsort((i, -j, k)) if grouped else np.lexsort((j, i))
    if direction == "conventional":
        return np.lexsort((-i, j, -k)) if grouped else np.lexsort((j, i))[::-1].copy()
    raise ValueError(f"unknown direction {direction!r}")


@dataclass
class OverlapBlock:
    """The 2b x b block handed from one worker's chase to the next (bulge.py:144-167)."""

    values: np.ndarray
    offset: int
    b: int

    def __post_init__(self):
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)
        if self.values.shape != (2 * self.b, self.b):
            raise ValueError(f"overlap must be {2 * self.b} x {self.b}")

    @property
    def words(self) -> int:
        return 2 * self.b * self.b


def final_gemm(q_sb_block, q_d, counter: FlopCounter | None = None) -> np.ndarray:
    """One block of rows of Q = Q_sb Q_d on the DMMA GEMM (backtrans.py:317-322)."""
    if q_sb_block.shape[1] != q_d.shape[0]:
        raise ValueError("inner dimensions disagree")
    out = device.dgemm(q_sb_block, q_d)
    if counter is not None:
        counter.add("FinalMultiply", q_sb_block.shape[0] * q_d.shape[1] * q_d.shape[0])
    return out
