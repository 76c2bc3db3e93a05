"""End-to-end parity of the single-GPU EVD (pevd_syevd_device) against the oracle.

Bounds: eigenvalues |lam - lam_ref| <= 10 n eps ||A||_2 (north star); residual
||A Q - Q Lam||_F / (n ||A||_F) and orthogonality ||Q^T Q - I||_F / n <= 1e-15 for n <= 1024
(the reference's own acceptance bar, tests/test_acceptance.py:34-50), 1e-12 at larger n.
"""
import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu
EPS = np.finfo(np.float64).eps


def dev():
    from paper_2511_16174_b200 import device
    return device


def sym(n, seed):
    g = np.random.default_rng(seed).standard_normal((n, n))
    return (g + g.T) / 2


@pytest.mark.parametrize("n,b,order", [(2, 4, "pipelined"), (3, 2, "pipelined"), (40, 4, "pipelined"),
                                       (64, 8, "sequential"), (64, 8, "conventional"),
                                       (97, 7, "pipelined"), (256, 32, "pipelined"),
                                       (256, 32, "conventional"), (1024, 32, "pipelined"),
                                       (300, 40, "pipelined"), (300, 40, "conventional"),
                                       (700, 64, "pipelined"), (700, 64, "conventional"),
                                       (129, 33, "sequential"), (500, 48, "conventional"),
                                       (400, 56, "pipelined")])
def test_syevd_matches_oracle(n, b, order):
    a = sym(n, n + b)
    lam, q, st = dev().syevd(a, b, True, order)
    lam_o, q_o = orc.evd(a, b, True, "pipelined")
    nrm2 = np.abs(lam_o).max()
    np.testing.assert_allclose(lam, lam_o, atol=10 * n * EPS * nrm2)
    assert orc.backward_error(a, q, lam) <= 1e-15
    assert orc.orthogonality(q) <= 1e-15


def test_values_only_equals_vectors_run():
    a = sym(300, 5)
    lam1, q, _ = dev().syevd(a, 32, True)
    lam2, q2, _ = dev().syevd(a, 32, False)
    assert q2 is None
    np.testing.assert_allclose(lam1, lam2, atol=1e-13 * np.abs(lam1).max())


def test_reruns_bitwise_identical():
    a = sym(500, 9)
    l1, q1, _ = dev().syevd(a, 32, True)
    l2, q2, _ = dev().syevd(a, 32, True)
    np.testing.assert_array_equal(l1, l2)
    np.testing.assert_array_equal(q1, q2)


@pytest.mark.parametrize("n", [2048, 4096])
def test_syevd_large_residual(n):
    a = sym(n, n)
    lam, q, st = dev().syevd(a, 32, True)
    assert orc.backward_error(a, q, lam) <= 1e-15
    assert orc.orthogonality(q) <= 1e-15
    lam_np = np.linalg.eigvalsh(a)
    np.testing.assert_allclose(lam, lam_np, atol=10 * n * EPS * np.abs(lam_np).max())


@pytest.mark.parametrize("order", ["pipelined", "sequential", "conventional"])
def test_padded_leading_dimensions(order):
    """lda = n + 7 and ldq = n + 3: the Y staircase SBR leaves in A is read back with lda by
    every SBR-Back path, and Q is written with its own stride (padding untouched)."""
    import ctypes
    import torch
    from paper_2511_16174_b200 import _lib
    L = _lib.load()
    n, b, lda, ldq = 300, 32, 307, 303
    a = sym(n, 77)
    oc = _lib.ORDER_CODES[order]
    A = torch.full((n, lda), 1e300, dtype=torch.float64, device="cuda")  # column-major, padded
    A[:, :n] = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()
    Q = torch.full((n, ldq), -7.0, dtype=torch.float64, device="cuda")
    lam = torch.empty(n, dtype=torch.float64, device="cuda")
    ws = torch.empty(L.pevd_syevd_workspace_bytes(n, b, 1, oc), dtype=torch.uint8, device="cuda")
    P = ctypes.c_void_p
    rc = L.pevd_syevd_device(n, b, P(A.data_ptr()), lda, P(lam.data_ptr()), P(Q.data_ptr()), ldq,
                             1, oc, P(ws.data_ptr()), ws.numel(),
                             P(torch.cuda.current_stream().cuda_stream), ctypes.byref(_lib.PevdStats()))
    _lib.check(rc, "pevd_syevd_device")
    q = np.asfortranarray(Q[:, :n].cpu().numpy().T)
    assert np.all(Q[:, n:].cpu().numpy() == -7.0)
    lam_h = lam.cpu().numpy()
    assert orc.backward_error(a, q, lam_h) <= 1e-15
    assert orc.orthogonality(q) <= 1e-15


def _device_run(a, b, order, poison_upper=False):
    """pevd_syevd_device on a column-major device copy of `a` (optionally with NaN in the
    strictly upper triangle): (lam, Q column-major as a Fortran array)."""
    import ctypes
    import torch
    from paper_2511_16174_b200 import _lib
    L = _lib.load()
    n = a.shape[0]
    oc = _lib.ORDER_CODES[order]
    A = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()  # rows of A^T = columns of A
    if poison_upper:
        iu = torch.triu_indices(n, n, 1)
        A[iu[1], iu[0]] = float("nan")                      # A[r, c] for r < c, column-major
    Q = torch.empty((n, n), dtype=torch.float64, device="cuda")
    lam = torch.empty(n, dtype=torch.float64, device="cuda")
    ws = torch.empty(L.pevd_syevd_workspace_bytes(n, b, 1, oc), dtype=torch.uint8, device="cuda")
    P = ctypes.c_void_p
    rc = L.pevd_syevd_device(n, b, P(A.data_ptr()), n, P(lam.data_ptr()), P(Q.data_ptr()), n, 1,
                             oc, P(ws.data_ptr()), ws.numel(),
                             P(torch.cuda.current_stream().cuda_stream), None)
    _lib.check(rc, "pevd_syevd_device")
    return lam.cpu().numpy(), np.asfortranarray(Q.cpu().numpy().T)


@pytest.mark.parametrize("order,b", [("conventional", 32), ("conventional", 12),
                                     ("pipelined", 32), ("sequential", 16)])
def test_strict_upper_triangle_never_read(order, b):
    """include/pevd.h: only the lower triangle of A is read -- the contract pevd_syevd's
    lower-trapezoid upload relies on.  NaN above the diagonal changes nothing, bit for bit."""
    a = sym(600, 41)
    l1, q1 = _device_run(a, b, order)
    l2, q2 = _device_run(a, b, order, poison_upper=True)
    np.testing.assert_array_equal(l1, l2)
    np.testing.assert_array_equal(q1, q2)


@pytest.mark.parametrize("n,order,pinned", [(700, "conventional", True),
                                            (700, "pipelined", False),
                                            (4500, "conventional", True),
                                            (4500, "conventional", False)])
def test_host_entry_point(n, order, pinned):
    """pevd_syevd (HOST buffers): lower-trapezoid upload, Q delivered slab by slab (n >= 4096
    runs SBR-Back in four column slabs whose copies overlap the next slab), pinned buffers by
    the copy engines, pageable ones through the native staging threads.  Same eigenpairs as the
    device entry point; the padding of Q (ldq > n) is left alone."""
    import ctypes
    import torch
    from paper_2511_16174_b200 import _lib
    L = _lib.load()
    b = 32
    a = sym(n, n + 3)
    lda, ldq = n + 5, n + 2
    if pinned:
        A = torch.zeros((n, lda), dtype=torch.float64, pin_memory=True)
        Qh = torch.full((n, ldq), -3.0, dtype=torch.float64, pin_memory=True)
        lam = torch.empty(n, dtype=torch.float64, pin_memory=True)
        A[:, :n] = torch.from_numpy(np.ascontiguousarray(a.T))
        A_np, Q_np, lam_np = A.numpy(), Qh.numpy(), lam.numpy()
    else:
        A_np = np.zeros((n, lda))
        A_np[:, :n] = a.T
        Q_np = np.full((n, ldq), -3.0)
        lam_np = np.empty(n)
    P = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    st = _lib.PevdStats()
    rc = L.pevd_syevd(n, b, P(A_np), lda, P(lam_np), P(Q_np), ldq, 1, _lib.ORDER_CODES[order],
                      ctypes.byref(st))
    _lib.check(rc, "pevd_syevd")
    assert np.all(Q_np[:, n:] == -3.0)
    q = np.asfortranarray(Q_np[:, :n].T)
    l_dev, q_dev = _device_run(a, b, order)
    np.testing.assert_allclose(lam_np, l_dev, atol=1e-13 * np.abs(l_dev).max())
    np.testing.assert_allclose(q, q_dev, atol=1e-11)
    assert orc.backward_error(a, q, lam_np) <= (1e-15 if n <= 1024 else 1e-12)
    assert orc.orthogonality(q) <= (1e-15 if n <= 1024 else 1e-12)
    assert st.sbr_back_ms[1] > 0


def _structured_cases():
    rng = np.random.default_rng(2024)
    n = 333
    yield "zero", np.zeros((n, n))
    yield "identity", np.eye(n)
    yield "diagonal", np.diag(rng.standard_normal(n))
    t = np.diag(rng.standard_normal(n)) + np.diag(rng.standard_normal(n - 1), 1)
    yield "tridiagonal", t + np.triu(t, 1).T
    u = rng.standard_normal(n)
    yield "rank1", np.outer(u, u)
    v = rng.standard_normal(n)
    v /= np.linalg.norm(v)
    yield "reflection", np.eye(n) - 2.0 * np.outer(v, v)     # eigenvalues -1 (once), +1 (n-1)
    blk = np.zeros((n, n))
    for s0 in range(0, n, 50):                               # decoupled blocks: exact zeros
        s1 = min(n, s0 + 50)
        g = rng.standard_normal((s1 - s0, s1 - s0))
        blk[s0:s1, s0:s1] = g + g.T
    yield "block_diagonal", blk
    g = rng.standard_normal((n, n))
    yield "tiny_scale", (g + g.T) * 1e-150
    yield "large_scale", (g + g.T) * 1e150
    for m in (33, 34, 65):                                   # n = b+1, b+2, 2b+1
        g = rng.standard_normal((m, m))
        yield f"n{m}", g + g.T


@pytest.mark.parametrize("case", list(_structured_cases()), ids=lambda c: c[0])
@pytest.mark.parametrize("order", ["pipelined", "conventional"])
def test_structured_inputs(case, order):
    """Inputs whose reductions hit the degenerate paths: zero columns below the band (tau = 0),
    an input that is already banded, exactly repeated eigenvalues (full deflation in the
    divide and conquer), decoupled blocks, extreme but representable scales, and n just above
    the bandwidth.  Bars as the reference's acceptance test (test_acceptance.py:34-50)."""
    name, a = case
    n = a.shape[0]
    lam, q, _ = dev().syevd(a, 32, True, order)
    lam_np = np.linalg.eigvalsh(a)
    nrm = np.abs(lam_np).max()
    assert np.all(np.diff(lam) >= 0)
    np.testing.assert_allclose(lam, lam_np, atol=10 * n * EPS * nrm)
    assert orc.backward_error(a, q, lam) <= 1e-15
    assert orc.orthogonality(q) <= 1e-15
    if name == "zero":
        np.testing.assert_array_equal(lam, np.zeros(n))


def test_bandwidth_above_64_rejected():
    """b <= 64 runs on the device kernels (multiples of 8 on the DMMA BC-Back, the rest on
    the generic paths); wider bands raise ValueError, as pipeline.py:57-82 does for bad configs."""
    import paper_2511_16174_b200 as pkg
    a = sym(200, 3)
    with pytest.raises(ValueError, match="64"):
        pkg.run(a, pkg.PipelineConfig(workers=1, b=65))


@pytest.mark.parametrize("n", [1, 2, 3, 40])
@pytest.mark.parametrize("want_vectors", [0, 1])
def test_host_entry_small_and_values_only(n, want_vectors):
    """pevd_syevd / pevd_syevd_checked on tiny sizes and without vectors (Q may be NULL), and
    the checked entry's ValueError on an asymmetric input before any reduction."""
    import ctypes
    from paper_2511_16174_b200 import _lib
    L = _lib.load()
    a = sym(n, 90 + n)
    af = np.asfortranarray(a)
    lam = np.empty(n)
    q = np.empty((n, n), order="F") if want_vectors else None
    vp = lambda x: x.ctypes.data_as(ctypes.c_void_p) if x is not None else None  # noqa: E731
    for checked in (False, True):
        if checked:
            rc = L.pevd_syevd_checked(n, 32, vp(af), n, vp(lam), vp(q), n, want_vectors, 2, 1e-13,
                                      0, None)
        else:
            rc = L.pevd_syevd(n, 32, vp(af), n, vp(lam), vp(q), n, want_vectors, 2, None)
        _lib.check(rc, "pevd_syevd")
        lam_np = np.linalg.eigvalsh(a)
        np.testing.assert_allclose(lam, lam_np, atol=10 * n * EPS * max(1.0, np.abs(lam_np).max()))
        if want_vectors:
            assert orc.backward_error(a, q, lam) <= 1e-15
            assert orc.orthogonality(q) <= 1e-15
    if n >= 2:
        bad = af.copy(order="F")
        bad[n - 1, 0] += 1e-3
        rc = L.pevd_syevd_checked(n, 32, vp(bad), n, vp(lam), vp(q), n, want_vectors, 2, 1e-13,
                                  0, None)
        assert rc == _lib.PEVD_ERR_VALUE
        assert "asymmetry" in L.pevd_last_error().decode()


@pytest.mark.parametrize("n,order,pinned", [(600, "pipelined", False), (4500, "pipelined", True),
                                            (4500, "sequential", False)])
def test_host_entry_row_major_q(n, order, pinned):
    """pipelined / sequential orders with q_row_major = 1: the final GEMM forms Q^T in column
    slabs streamed to the host, so the host buffer holds Q C-ordered (pipeline.py:503); the same
    eigenpairs as the device entry point, and conventional order refuses row-major output."""
    import ctypes
    import torch
    from paper_2511_16174_b200 import _lib
    L = _lib.load()
    a = sym(n, 7 * n)
    af = np.asfortranarray(a)
    lam = np.empty(n)
    if pinned:
        qt = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        q = qt.numpy()
    else:
        q = np.empty((n, n))                                   # C order
    vp = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    oc = _lib.ORDER_CODES[order]
    _lib.check(L.pevd_syevd_checked(n, 32, vp(af), n, vp(lam), vp(q), n, 1, oc, -1.0, 1, None),
               "pevd_syevd_checked")
    l_dev, q_dev = _device_run(a, 32, order)
    np.testing.assert_allclose(lam, l_dev, atol=1e-13 * np.abs(l_dev).max())
    np.testing.assert_allclose(q, q_dev, atol=1e-11)        # q (C order) is Q itself
    assert orc.backward_error(a, q, lam) <= (1e-15 if n <= 1024 else 1e-12)
    rc = L.pevd_syevd_checked(n, 32, vp(af), n, vp(lam), vp(q), n, 1, 2, -1.0, 1, None)
    assert rc == _lib.PEVD_ERR_VALUE
