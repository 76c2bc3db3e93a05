"""Per-stage parity of the CUDA path (libpevd.so via the C ABI) against the CPU oracle.

Tolerances: the oracle is pinned bit-exact to the reference (tests/test_oracle.py); the device
kernels reorder floating-point sums, so stage outputs are compared at 1e-12..1e-13 relative to
the problem scale, the bounds the reference's own tests use (tests/test_sbr.py:94-125,
tests/test_bulge.py:23-48, tests/test_tridiag.py:22-44).
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


@pytest.mark.parametrize("m,n,k,ta,tb", [(1, 1, 1, 0, 0), (37, 29, 53, 0, 0), (130, 70, 300, 1, 0),
                                         (64, 200, 17, 0, 1), (257, 33, 1000, 1, 1),
                                         (300, 32, 5000, 1, 0), (32, 32, 20000, 1, 0),
                                         (1000, 900, 64, 0, 1),
                                         # deep split-K of tiny outputs (W^T AW) and t = P2^T W
                                         (29, 31, 30001, 1, 0), (32, 32, 49152, 1, 0),
                                         (960, 32, 49152, 1, 0)])
def test_dgemm_matches_numpy(m, n, k, ta, tb):
    rng = np.random.default_rng(m * 7 + n)
    a = rng.standard_normal((k, m) if ta else (m, k))
    b = rng.standard_normal((n, k) if tb else (k, n))
    c = rng.standard_normal((m, n))
    got = dev().dgemm(a, b, alpha=1.5, beta=-0.5, c=c, trans_a=bool(ta), trans_b=bool(tb))
    want = 1.5 * ((a.T if ta else a) @ (b.T if tb else b)) - 0.5 * c
    np.testing.assert_allclose(got, want, atol=1e-12 * np.sqrt(k) * 4, rtol=0)


@pytest.mark.parametrize("m,k", [(8, 8), (40, 8), (300, 32), (1000, 32), (5000, 17), (20000, 32),
                                 (4097, 31), (49152, 32),  # one-pass kernel, ragged / full grid
                                 (100, 33), (700, 48), (3000, 64), (40000, 64)])
def test_panel_qr_matches_oracle(m, k):
    p = np.random.default_rng(m + k).standard_normal((m, k))
    R, Y, W, T = dev().panel_qr(p)
    pp = p.copy(order="F")
    Wo, Yo = orc.panel_qr(pp)
    np.testing.assert_allclose(Y, Yo, atol=1e-12)
    np.testing.assert_allclose(W, Wo, atol=1e-12)
    np.testing.assert_allclose(np.triu(R), np.triu(pp[:k]), atol=1e-11 * np.abs(p).max())
    np.testing.assert_allclose(W, Y @ T, atol=1e-13)
    q = np.eye(m) - W @ Y.T if m <= 2000 else None
    if q is not None:
        np.testing.assert_allclose(q.T @ p, np.vstack([np.triu(R), np.zeros((m - k, k))]),
                                   atol=1e-12 * np.abs(p).max() * np.sqrt(m))


@pytest.mark.parametrize("n,b", [(12, 4), (11, 4), (64, 8), (91, 7), (200, 32), (513, 32), (1024, 32),
                                 (300, 40), (600, 64)])
def test_sbr_band_matches_oracle(n, b):
    a = sym(n, n + b)
    bands, ystair, tall = dev().sbr(a, b)
    bands_o, panels = orc.sbr_reduce(a, b)
    np.testing.assert_allclose(bands, bands_o, atol=1e-12 * np.linalg.norm(a))
    # the explicit-Y staircase holds every panel's Y
    for x, (c0, W, Y) in enumerate(panels):
        t0 = c0 + b
        np.testing.assert_allclose(ystair[t0:, c0:c0 + Y.shape[1]], Y, atol=1e-11)


@pytest.mark.parametrize("n,b", [(10, 2), (24, 3), (40, 4), (64, 8), (100, 16), (130, 32), (700, 32),
                                 (80, 33), (500, 48), (900, 64)])
def test_bc_matches_oracle(n, b):
    rng = np.random.default_rng(n * b)
    a = rng.standard_normal((n, n))
    a = np.tril(np.triu((a + a.T) / 2, -b), b)
    bands = orc.band_from_dense(a, b)
    d, e, tau, V = dev().bc(bands)
    do, eo, refl = orc.bc_reduce(bands)
    scale = np.linalg.norm(a)
    np.testing.assert_allclose(d, do, atol=1e-12 * scale)
    np.testing.assert_allclose(np.abs(e), np.abs(eo), atol=1e-12 * scale)
    got = dev().slots_to_reference(n, b, tau, V)
    assert len(got["tau"]) == len(refl["tau"])
    np.testing.assert_array_equal(got["i"], refl["i"])
    np.testing.assert_array_equal(got["j"], refl["j"])
    np.testing.assert_allclose(got["tau"], refl["tau"], atol=1e-10)
    np.testing.assert_allclose(got["v"], refl["v"], atol=1e-9)


def _tridiag_cases():
    rng = np.random.default_rng(7)
    yield "rand40", rng.standard_normal(40), rng.standard_normal(39)
    yield "rand300", rng.standard_normal(300), rng.standard_normal(299)
    yield "rand2000", rng.standard_normal(2000), rng.standard_normal(1999)
    yield "one", np.array([2.5]), np.zeros(0)
    yield "two", np.array([2.0, 0.0]), np.array([1.0])
    yield "diag", np.array([3.0, -1.0, 2.0]), np.zeros(2)
    n = 500
    yield "wilkinson", np.abs(np.arange(n) - (n - 1) / 2.0), np.ones(n - 1)
    yield "clustered", np.r_[np.full(n - 1, 1e-2), 1e6], np.full(n - 1, 1e-9)
    yield "toeplitz", np.full(777, 2.0), np.full(776, -1.0)
    yield "graded", 10.0 ** -np.arange(60.0) * 0 + np.linspace(1, 2, 60), 1e-8 * np.ones(59)
    yield "zeros", np.zeros(100), np.zeros(99)
    yield "glued", np.tile(np.array([1.0, 2.0, 3.0, 4.0]), 64), np.r_[np.tile([1.0, 1.0, 1.0, 1e-12], 63), [1.0, 1.0, 1.0]]


@pytest.mark.parametrize("case", list(_tridiag_cases()), ids=lambda c: c[0])
def test_stedc_matches_reference_solver(case):
    name, d, e = case
    n = len(d)
    lam, q = dev().stedc(d, e)
    t = np.diag(d) + (np.diag(e, 1) + np.diag(e, -1) if n > 1 else 0)
    nrm = max(1.0, np.abs(np.linalg.eigvalsh(t)).max())
    lam_o, q_o = orc.tridiag_eig(d, e, want_vectors=True)
    # eigenvalues: |lam - lam_ref| <= 10 n eps ||T||_2 (north-star bound), ascending
    assert np.all(np.diff(lam) >= 0)
    np.testing.assert_allclose(lam, lam_o, atol=10 * n * EPS * nrm)
    # residual and orthogonality (reference tests/test_tridiag.py:35-44 use 1e-13)
    np.testing.assert_allclose(t @ q, q * lam, atol=1e-13 * nrm * max(1, np.sqrt(n) / 10))
    np.testing.assert_allclose(q.T @ q, np.eye(n), atol=1e-13 * max(1, np.sqrt(n) / 10))
    # sign convention (tridiag.py:325-333)
    for j in range(n):
        col = q[:, j]
        assert col[np.argmax(np.abs(col))] > 0


@pytest.mark.parametrize("n,b", [(24, 3), (64, 8), (130, 32), (500, 32), (701, 32), (333, 8),
                                 (400, 16), (515, 24), (257, 12), (300, 40), (350, 48),
                                 (200, 56), (400, 64), (300, 44)])
def test_bc_back_matches_oracle(n, b):
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n))
    a = np.tril(np.triu((a + a.T) / 2, -b), b)
    bands = orc.band_from_dense(a, b)
    d, e, tau, V = dev().bc(bands)
    _, _, refl = orc.bc_reduce(bands)
    x = rng.standard_normal((37, n))
    got = dev().bc_back_right(n, b, tau, V, x)
    want = orc.bc_back_apply(refl, x.T, "reordered").T
    np.testing.assert_allclose(got, want, atol=1e-11)
    y = rng.standard_normal((n, 5))
    got = dev().bc_back_left(n, b, tau, V, y)
    want = orc.bc_back_apply(refl, y, "conventional")
    np.testing.assert_allclose(got, want, atol=1e-11)


@pytest.mark.parametrize("n,b", [(12, 4), (91, 7), (300, 32), (1000, 32)])
def test_sbr_back_form_matches_oracle(n, b):
    a = sym(n, 3 * n)
    bands, ystair, tall = dev().sbr(a, b)
    qs = dev().sbr_back_form(n, b, ystair, tall)
    _, panels = orc.sbr_reduce(a, b)
    qs_o = orc.sbr_back_accumulate(n, panels, (0, n))
    np.testing.assert_allclose(qs, qs_o, atol=1e-12 * np.sqrt(n))
    band_dense = orc.band_to_dense(bands)
    np.testing.assert_allclose(qs.T @ a @ qs, band_dense, atol=1e-12 * np.linalg.norm(a))


@pytest.mark.parametrize("n,c0,c1", [(2000, 600, 1400), (4096, 0, 1000), (4096, 3000, 4096),
                                     (700, 350, 351)])
def test_stedc_column_range_matches_full(n, c0, c1):
    """pevd_stedc_cols forms exactly the wanted eigenvector columns of the full D&C (the top
    merge GEMM restricted to them), bit for bit; all eigenvalues; the rest of Q stays zero."""
    import ctypes
    import torch
    from paper_2511_16174_b200 import _lib
    L = _lib.load()
    rng = np.random.default_rng(n + c0)
    d0 = rng.standard_normal(n)
    e0 = rng.standard_normal(n - 1)
    P = ctypes.c_void_p
    s = P(torch.cuda.current_stream().cuda_stream)
    out = []
    for cols in (None, (c0, c1)):
        d = torch.from_numpy(d0.copy()).cuda()
        e = torch.from_numpy(np.append(e0, 0.0)).cuda()
        Q = torch.full((n, n), 7.0, dtype=torch.float64, device="cuda")
        ws = torch.empty(L.pevd_stedc_workspace_bytes(n), dtype=torch.uint8, device="cuda")
        if cols is None:
            rc = L.pevd_stedc(n, P(d.data_ptr()), P(e.data_ptr()), P(Q.data_ptr()), n,
                              P(ws.data_ptr()), s)
        else:
            rc = L.pevd_stedc_cols(n, P(d.data_ptr()), P(e.data_ptr()), P(Q.data_ptr()), n,
                                   cols[0], cols[1], P(ws.data_ptr()), s)
        _lib.check(rc, "stedc")
        out.append((d.cpu().numpy(), Q.cpu().numpy().T))
    (lam_f, q_f), (lam_c, q_c) = out
    np.testing.assert_array_equal(lam_c, lam_f)
    np.testing.assert_array_equal(q_c[:, c0:c1], q_f[:, c0:c1])
