"""Per-stage device operations over the C ABI (include/pevd.h).

Each function mirrors one reference function (file:line in the docstring) and runs it on the
GPU through libpevd.so.  Matrices cross the boundary column-major (Fortran order): a
column-major n x m matrix lives in a torch tensor of shape (m, n).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


def _torch():
    return _lib.require_cuda()


def _stream():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def to_dev(a: np.ndarray):
    """numpy matrix -> column-major device tensor (shape (cols, rows))."""
    torch = _torch()
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        return torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return torch.from_numpy(np.ascontiguousarray(a.T)).cuda()


def from_dev(t, rows: int | None = None) -> np.ndarray:
    """column-major device tensor -> numpy (Fortran-ordered) matrix."""
    h = t.detach().cpu().numpy()
    if h.ndim == 1:
        return h
    return np.asfortranarray(h.T)


def empty(rows: int, cols: int = 0):
    torch = _torch()
    if cols == 0:
        return torch.empty(max(rows, 1), dtype=torch.float64, device="cuda")
    return torch.empty((max(cols, 1), max(rows, 1)), dtype=torch.float64, device="cuda")


def workspace(nbytes: int):
    torch = _torch()
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device="cuda")


def _p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def dgemm(a, b, alpha=1.0, beta=0.0, c=None, trans_a=False, trans_b=False):
    """C = alpha op(A) op(B) + beta C on the FP64 DMMA GEMM (core.py:309-319 matmul_counted)."""
    L = _lib.load()
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    m = a.shape[1] if trans_a else a.shape[0]
    k = a.shape[0] if trans_a else a.shape[1]
    n = b.shape[0] if trans_b else b.shape[1]
    da, db = to_dev(a), to_dev(b)
    dc = to_dev(c) if c is not None else empty(m, n)
    ws = workspace(8 << 20 * 1)
    rc = L.pevd_dgemm(int(trans_a), int(trans_b), m, n, k, alpha, _p(da), a.shape[0], _p(db),
                      b.shape[0], beta, _p(dc), m, _p(ws), ws.numel(), _stream())
    _lib.check(rc, "dgemm")
    return from_dev(dc)


def dsymm_lower(a, b):
    """A B with A symmetric, read from its lower triangle only (pevd_dsymm_lower)."""
    L = _lib.load()
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    m, n = a.shape[0], b.shape[1]
    da, db = to_dev(a), to_dev(b)
    dc = empty(m, n)
    ws = workspace(8 << 20)
    rc = L.pevd_dsymm_lower(m, n, 1.0, _p(da), m, _p(db), m, 0.0, _p(dc), m, _p(ws), ws.numel(),
                            _stream())
    _lib.check(rc, "dsymm_lower")
    return from_dev(dc)


def panel_qr(panel):
    """Householder panel QR (sbr.py:69-116) -> (R, Y, W, T); Q = I - W Y^T, Q^T P = R."""
    L = _lib.load()
    p = np.asarray(panel, dtype=np.float64)
    m, k = p.shape
    dp = to_dev(p)
    dr, dy, dw, dt = empty(k, k), empty(m, k), empty(m, k), empty(k, k)
    ws = workspace(L.pevd_panel_qr_workspace_bytes())
    rc = L.pevd_panel_qr(m, k, _p(dp), m, _p(dr), _p(dy), m, _p(dw), m, _p(dt), _p(ws), _stream())
    _lib.check(rc, "panel_qr")
    return from_dev(dr), from_dev(dy), from_dev(dw), from_dev(dt)


def sbr(a, b):
    """Band reduction (sbr.py:155-188) -> (bands (b+1, n), Y staircase (n, n), Tall flat)."""
    L = _lib.load()
    a = np.asarray(a, dtype=np.float64)
    n = a.shape[0]
    da = to_dev(a)
    torch = _torch()
    bands = torch.empty((b + 1) * n, dtype=torch.float64, device="cuda")
    rounds = max(1, -(-(n - b) // b))
    tall = torch.zeros(rounds * b * b, dtype=torch.float64, device="cuda")
    ws = workspace(L.pevd_sbr_workspace_bytes(n, b))
    rc = L.pevd_sbr(n, b, _p(da), n, _p(bands), _p(tall), _p(ws), _stream())
    _lib.check(rc, "sbr")
    # tall: flat, panel x's T (pw x pw, column-major, ld pw) at offset x * b * b
    return bands.cpu().numpy().reshape(b + 1, n), from_dev(da), tall.cpu().numpy()


def bc(bands, want_reflectors=True):
    """Bulge chasing (bulge.py:299-309) -> (d, e, tau slots, V slots (nslots x vld))."""
    L = _lib.load()
    bands = np.ascontiguousarray(bands, dtype=np.float64)
    b = bands.shape[0] - 1
    n = bands.shape[1]
    torch = _torch()
    dbands = torch.from_numpy(bands.reshape(-1)).cuda()
    d, e = empty(n), empty(max(n - 1, 1))
    nref = L.pevd_bc_num_reflectors(n, b)
    vld = ((b + 7) // 8) * 8
    tau = torch.zeros(max(nref, 1), dtype=torch.float64, device="cuda") if want_reflectors else None
    V = torch.zeros(max(nref, 1) * vld, dtype=torch.float64, device="cuda") if want_reflectors else None
    ws = workspace(L.pevd_bc_workspace_bytes(n, b))
    rc = L.pevd_bc(n, b, _p(dbands), _p(d), _p(e), _p(tau), _p(V), vld, _p(ws), _stream())
    _lib.check(rc, "bc")
    out_tau = tau.cpu().numpy()[:nref] if want_reflectors else None
    out_v = V.cpu().numpy()[: nref * vld].reshape(nref, vld) if want_reflectors else None
    return d.cpu().numpy()[:n], e.cpu().numpy()[: n - 1], out_tau, out_v


def bc_partition(bands, b: int, sweep_end: int):
    """Partition chase (bulge.py:348-385) on a band of semi-bandwidth bw = bands.shape[0] - 1
    <= 2b: sweeps [0, sweep_end) -> ((2b+1) x n band afterwards, tau slots, V slots)."""
    L = _lib.load()
    bands = np.ascontiguousarray(bands, dtype=np.float64)
    bw, n = bands.shape[0] - 1, bands.shape[1]
    torch = _torch()
    dbands = torch.from_numpy(bands.reshape(-1)).cuda()
    out = torch.zeros((2 * b + 1) * n, dtype=torch.float64, device="cuda")
    nref = L.pevd_bc_num_reflectors(n, b)
    vld = ((b + 7) // 8) * 8
    tau = torch.zeros(max(nref, 1), dtype=torch.float64, device="cuda")
    V = torch.zeros(max(nref, 1) * vld, dtype=torch.float64, device="cuda")
    ws = workspace(L.pevd_bc_workspace_bytes(n, b))
    rc = L.pevd_bc_partition(n, b, bw, _p(dbands), int(sweep_end), _p(out), _p(tau), _p(V), vld,
                             _p(ws), _stream())
    _lib.check(rc, "bc_partition")
    return (out.cpu().numpy().reshape(2 * b + 1, n), tau.cpu().numpy()[:nref],
            V.cpu().numpy()[: nref * vld].reshape(nref, vld))


def slot_offset(n: int, b: int, j: int) -> int:
    """Fixed reflector slot layout of pevd_bc: slot(i, j) = offset(j) + i (include/pevd.h)."""
    return j * (n - 2) - b * j * (j - 1) // 2


def slots_to_reference(n: int, b: int, tau, V):
    """Fixed slots -> the reference BulgeReflectorSet arrays (bulge.py:33-68): only recorded
    reflectors (tau != 0), canonical order (chase step j outer, sweep i inner)."""
    stride = ((b + 7) // 8) * 8
    tau = np.asarray(tau).reshape(-1)
    V = np.asarray(V).reshape(len(tau), -1) if len(tau) else np.zeros((0, stride))
    js, is_ = [], []
    j = 0
    while n - 2 - j * b > 0:        # slot(i, j) = offset(j) + i, i < n - 2 - j b
        cnt = n - 2 - j * b
        js.append(np.full(cnt, j, dtype=np.int64))
        is_.append(np.arange(cnt, dtype=np.int64))
        j += 1
    jj = np.concatenate(js) if js else np.zeros(0, np.int64)
    ii = np.concatenate(is_) if is_ else np.zeros(0, np.int64)
    keep = np.nonzero(tau[: len(jj)] != 0.0)[0]       # slot order is already (j, i) order
    r0 = ii[keep] + 1 + jj[keep] * b
    v = np.zeros((len(keep), stride))
    w = min(stride, V.shape[1]) if len(keep) else 0
    if len(keep):
        v[:, :w] = V[keep, :w]
    return dict(i=ii[keep], j=jj[keep], row0=r0, len=np.minimum(b, n - r0),
                tau=tau[keep].copy(), v=v)


def stedc(d, e):
    """Tridiagonal divide and conquer (replaces tridiag_eig, tridiag.py:298-334) -> (lam, Q)."""
    L = _lib.load()
    d = np.asarray(d, dtype=np.float64)
    n = d.shape[0]
    dd = to_dev(d)
    de = to_dev(np.asarray(e, dtype=np.float64) if n > 1 else np.zeros(1))
    q = empty(n, n)
    ws = workspace(L.pevd_stedc_workspace_bytes(n))
    rc = L.pevd_stedc(n, _p(dd), _p(de), _p(q), n, _p(ws), _stream())
    if rc == _lib.PEVD_ERR_CONVERGE:
        raise RuntimeError(L.pevd_last_error().decode())
    _lib.check(rc, "stedc")
    return dd.cpu().numpy()[:n], from_dev(q)


def sbr_back_form(n, b, ystair, tall):
    """Q_s = prod (I - Y_x T_x Y_x^T) (backtrans.py:128-146, all columns)."""
    L = _lib.load()
    torch = _torch()
    dy = to_dev(ystair)
    dt = torch.from_numpy(np.ascontiguousarray(tall, dtype=np.float64).reshape(-1)).cuda()
    q = empty(n, n)
    ws = workspace(L.pevd_sbr_back_workspace_bytes(n, b))
    rc = L.pevd_sbr_back_form(n, b, _p(dy), n, _p(dt), _p(q), n, _p(ws), _stream())
    _lib.check(rc, "sbr_back_form")
    return from_dev(q)


def t_block(tall, x: int, b: int, pw: int) -> np.ndarray:
    """Panel x's T factor (pw x pw) out of the flat Tall array."""
    o = x * b * b
    return np.asarray(tall).reshape(-1)[o:o + pw * pw].reshape(pw, pw).T.copy()


def bc_back_right(n, b, tau, V, x):
    """X <- X Q_b (reordered BC-Back, backtrans.py:277-310, transposed)."""
    L = _lib.load()
    torch = _torch()
    x = np.asarray(x, dtype=np.float64)
    vld = V.shape[1]
    dt = torch.from_numpy(np.ascontiguousarray(tau)).cuda()
    dv = torch.from_numpy(np.ascontiguousarray(V).reshape(-1)).cuda()
    dx = to_dev(x)
    ws = workspace(L.pevd_bc_back_workspace_bytes(n, x.shape[0], b))
    rc = L.pevd_bc_back_right(n, b, _p(dt), _p(dv), vld, _p(dx), x.shape[0], x.shape[0], _p(ws),
                              _stream())
    _lib.check(rc, "bc_back_right")
    return from_dev(dx)


def bc_back_left(n, b, tau, V, x):
    """X <- Q_b X (conventional BC-Back, backtrans.py:277-310)."""
    L = _lib.load()
    torch = _torch()
    x = np.asarray(x, dtype=np.float64)
    vld = V.shape[1]
    dt = torch.from_numpy(np.ascontiguousarray(tau)).cuda()
    dv = torch.from_numpy(np.ascontiguousarray(V).reshape(-1)).cuda()
    dx = to_dev(x)
    ws = workspace(L.pevd_bc_back_workspace_bytes(n, x.shape[1], b))
    rc = L.pevd_bc_back_left(n, b, _p(dt), _p(dv), vld, _p(dx), x.shape[0], x.shape[1], _p(ws),
                             _stream())
    _lib.check(rc, "bc_back_left")
    return from_dev(dx)


STAGED_MIN_BYTES = 256 << 20  # larger host <-> device copies go through pinned staging
STAGE_THREADS = 8
STAGE_CHUNK = 1 << 22          # doubles per chunk (32 MB)


def _staged_copy(host: np.ndarray, dev, to_device: bool):
    """Host <-> device copy of a contiguous numpy array through pinned staging buffers, several
    host threads at once (torch copies release the GIL).  A 19.3 GB pageable copy takes 3.6 s
    host -> device and 10.3 s device -> host (first-touch page faults, one thread) on the pool's
    B200 boxes; staged with 8 threads it is ~1.5 s (tools/h2d_probe.py)."""
    import threading
    torch = _torch()
    flat_h = torch.from_numpy(host.reshape(-1))
    flat_d = dev.view(-1)
    N = flat_h.numel()
    errs = []

    def work(tid):
        try:
            st = torch.cuda.Stream()
            bufs = [torch.empty(STAGE_CHUNK, dtype=torch.float64, pin_memory=True)
                    for _ in range(2)]
            evs = [None, None]
            k = 0
            for c0 in range(tid * STAGE_CHUNK, N, STAGE_THREADS * STAGE_CHUNK):
                c1 = min(N, c0 + STAGE_CHUNK)
                buf = bufs[k & 1][: c1 - c0]
                if evs[k & 1] is not None:
                    evs[k & 1].synchronize()
                with torch.cuda.stream(st):
                    if to_device:
                        buf.copy_(flat_h[c0:c1])
                        flat_d[c0:c1].copy_(buf, non_blocking=True)
                    else:
                        buf.copy_(flat_d[c0:c1], non_blocking=True)
                        st.synchronize()
                        flat_h[c0:c1].copy_(buf)
                    e = torch.cuda.Event()
                    e.record(st)
                    evs[k & 1] = e
                k += 1
            st.synchronize()
        except BaseException as exc:  # surfaced below
            errs.append(exc)

    torch.cuda.synchronize()
    th = [threading.Thread(target=work, args=(i,)) for i in range(STAGE_THREADS)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]


def _to_device(mem: np.ndarray):
    torch = _torch()
    if mem.nbytes < STAGED_MIN_BYTES:
        return torch.from_numpy(mem).cuda()
    out = torch.empty(mem.shape, dtype=torch.float64, device="cuda")
    _staged_copy(mem, out, True)
    return out


def _to_host(t) -> np.ndarray:
    if t.numel() * 8 < STAGED_MIN_BYTES:
        return t.cpu().numpy()
    out = np.empty(tuple(t.shape), dtype=np.float64)
    _staged_copy(out, t.contiguous(), False)
    return out


def syevd(a, b=32, want_vectors=True, order="pipelined", stats=None, check_sym=False,
          sym_tol=1e-13):
    """Whole single-GPU EVD through pevd_syevd_device: (lam, Q or None, PevdStats).

    The host array goes to the device without a host-side transpose: a Fortran-order array is
    A column-major, a C-order one is A^T column-major (the same matrix when symmetric).
    check_sym: the SymmetricMatrix test (core.py:75-84) runs on the device (pevd_asymmetry)
    instead of over the host copy.  Q comes back Fortran-ordered in conventional order and
    C-ordered otherwise (pipeline.py:495, 503) -- the device transposes, not the host.
    With vectors this is one native call (pevd_syevd_checked): the library moves the host
    buffers itself and overlaps Q's download with the last GEMMs."""
    L = _lib.load()
    torch = _torch()
    a = np.asarray(a, dtype=np.float64)
    n = a.shape[0]
    oc = _lib.ORDER_CODES[order]
    bb = max(1, min(b, n - 1)) if n > 1 else 1
    mem = a.T if a.flags.f_contiguous else np.ascontiguousarray(a)
    st = _lib.PevdStats() if stats is None else stats
    if want_vectors:
        # one native call: the upload (lower trapezoid, or all of A for the device symmetry
        # check) and Q's download slab by slab under the last GEMMs (SBR-Back in conventional
        # order, the final multiply otherwise) go through the library's own staging threads.
        # Q lands as the reference returns it: Fortran-ordered in conventional order, C-ordered
        # otherwise (pipeline.py:495, 503; the final GEMM then forms Q^T slab by slab)
        lam_h = np.empty(n)
        conv = order == "conventional"
        qh = np.empty((n, n), dtype=np.float64, order="F" if conv else "C")
        vp = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        rc = L.pevd_syevd_checked(n, bb, vp(mem), n, vp(lam_h), vp(qh), n, 1, oc,
                                  sym_tol if check_sym else -1.0, 0 if conv else 1,
                                  ctypes.byref(st))
        if rc == _lib.PEVD_ERR_CONVERGE:
            raise RuntimeError(L.pevd_last_error().decode())
        _lib.check(rc, "syevd")
        return lam_h, qh, st
    da = _to_device(mem)                  # (n, n): column-major A (or A^T)
    if check_sym:
        out = (ctypes.c_double * 2)()
        _lib.check(L.pevd_asymmetry(n, _p(da), n, out, _stream()), "asymmetry check")
        if out[0] > sym_tol * max(1.0, out[1]):
            raise ValueError(f"asymmetry {out[0]:.3e} exceeds tolerance")
    lam = empty(n)
    q = empty(n, n) if want_vectors else None
    ws = workspace(L.pevd_syevd_workspace_bytes(n, bb, int(want_vectors), oc))
    rc = L.pevd_syevd_device(n, bb, _p(da), n, _p(lam), _p(q), n, int(want_vectors), oc, _p(ws),
                             ws.numel(), _stream(), ctypes.byref(st))
    if rc == _lib.PEVD_ERR_CONVERGE:
        raise RuntimeError(L.pevd_last_error().decode())
    _lib.check(rc, "syevd")
    del ws, da
    qh = None
    if want_vectors:
        qt = torch.empty_like(q)                      # C order: transposed on the device
        _lib.check(L.pevd_transpose(n, n, _p(q), n, _p(qt), n, _stream()), "transpose")
        del q
        qh = _to_host(qt)
    return lam.cpu().numpy()[:n], qh, st


def syevd_multi(a, workers: int, b: int, col_ranges, back_ranges, want_vectors=True,
                order="pipelined", devices=None):
    """Blockwise EVD over `workers` cooperating devices in this process (pevd_syevd_multi: one
    host thread per worker, peer-to-peer transfers).  Workers map round-robin onto the visible
    GPUs; with fewer GPUs than workers, several workers share a device (same protocol, same
    messages, no extra parallelism).  Returns (lam, Q (Fortran order in conventional order,
    C order otherwise) or None, [PevdDistStats per worker])."""
    L = _lib.load()
    torch = _torch()
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    n = a.shape[0]
    G = int(workers)
    if devices is None:
        ngpu = torch.cuda.device_count()
        devices = [w % ngpu for w in range(G)]
    devs = (ctypes.c_int * G)(*devices)
    col_lo = (ctypes.c_int64 * (G + 1))(*([lo for lo, _ in col_ranges] + [n]))
    back_lo = (ctypes.c_int64 * (G + 1))(*([lo for lo, _ in back_ranges] + [n]))
    lam = np.empty(n, dtype=np.float64)
    q = None
    if want_vectors:
        q = np.empty((n, n), dtype=np.float64,
                     order="F" if order == "conventional" else "C")
    stats = (_lib.PevdDistStats * G)()
    keep = [_lib.new_dist_stats() for _ in range(G)]
    for w in range(G):
        stats[w] = keep[w]
    rc = L.pevd_syevd_multi(G, devs, n, b, a.ctypes.data_as(ctypes.c_void_p), n, col_lo, back_lo,
                            lam.ctypes.data_as(ctypes.c_void_p),
                            q.ctypes.data_as(ctypes.c_void_p) if q is not None else None,
                            int(want_vectors), _lib.ORDER_CODES[order], stats)
    if rc == _lib.PEVD_ERR_CONVERGE:
        raise RuntimeError(L.pevd_last_error().decode())
    _lib.check(rc, "syevd_multi")
    out = []
    for w in range(G):
        st = stats[w]
        st._ev, st._ms = keep[w]._ev, keep[w]._ms
        out.append(st)
    return lam, q, out
