"""Full-size parity through size-independent properties (BASELINE.json configs c2-c5 on one GPU).

The oracle cannot run at n = 8192-49152, so these tests check what the reference's own
acceptance tests check, on planted-spectrum matrices generated on the device
(paper_2511_16174_b200/matgen.py): the eigenvalues must equal the planted ones within the north
star's 10 n eps ||A||_2, and the eigenvectors must satisfy residual ||AQ - Q Lam||_F/(n||A||_F)
<= 1e-12 and orthogonality ||Q^T Q - I||_F/n <= 1e-12 (north star).  The clustered families
(Cluster0/Cluster1, config c5) drive the divide and conquer through near-total deflation.
"""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
EPS = np.finfo(np.float64).eps


def _evd(A, n, b, order):
    import torch
    from paper_2511_16174_b200 import _lib
    L = _lib.load()
    oc = _lib.ORDER_CODES[order]
    lam = torch.empty(n, dtype=torch.float64, device="cuda")
    Q = torch.empty((n, n), dtype=torch.float64, device="cuda")
    ws = torch.empty(L.pevd_syevd_workspace_bytes(n, b, 1, oc), dtype=torch.uint8, device="cuda")
    P = ctypes.c_void_p
    st = _lib.PevdStats()
    rc = L.pevd_syevd_device(n, b, P(A.data_ptr()), n, P(lam.data_ptr()), P(Q.data_ptr()), n, 1,
                             oc, P(ws.data_ptr()), ws.numel(),
                             P(torch.cuda.current_stream().cuda_stream), ctypes.byref(st))
    _lib.check(rc, "pevd_syevd_device")
    del ws
    torch.cuda.empty_cache()
    return lam, Q, st


@pytest.mark.parametrize("kind,n,order", [
    ("Normal", 49152, "conventional"),      # c4: the headline size
    ("Geometric", 8192, "pipelined"),       # c2
    ("Arithmetic", 8192, "sequential"),
    ("Cluster0", 16384, "conventional"),    # c5 family: one eigenvalue + a 16383-fold cluster
    ("Cluster1", 16384, "pipelined"),
    ("Uniform", 16384, "conventional"),
    ("Normal", 20001, "conventional"),      # ragged sizes: partial row blocks, groups, tiles
    ("Normal", 12345, "pipelined"),
    ("Normal", 9999, "sequential"),
])
def test_planted_spectrum(kind, n, order):
    import torch
    from paper_2511_16174_b200 import matgen
    spec = matgen.SpectrumSpec(kind, n, seed=n + 7)
    A, lam_true = matgen.generate(spec)
    lam, Q, st = _evd(A, n, 32, order)       # A is overwritten by the reduction
    lam_h = lam.cpu().numpy()
    nrm2 = float(np.abs(lam_true).max())
    err = float(np.abs(lam_h - lam_true).max())
    assert err <= 10 * n * EPS * nrm2, f"{kind} n={n}: |dlam| {err:.3e}"
    assert np.all(np.diff(lam_h) >= 0)
    A = matgen.planted(lam_true, seed=spec.seed, out=A)  # regenerate the input (deterministic)
    res, orth = matgen.accuracy(A, lam, Q)
    del A, Q
    torch.cuda.empty_cache()
    assert res <= 1e-12 and orth <= 1e-12, f"{kind} n={n}: residual {res:.2e}, ortho {orth:.2e}"


def test_planted_generator_is_exact_small():
    """The device generator's A really has the planted spectrum (numpy eigvalsh at n = 512)."""
    from paper_2511_16174_b200 import matgen
    spec = matgen.SpectrumSpec("Geometric", 512, cond=1e4, lambda_max=10.0, seed=3)
    A, lam = matgen.generate(spec, k=48)
    a = A.cpu().numpy().T
    assert np.abs(a - a.T).max() <= 1e-13 * 10.0
    np.testing.assert_allclose(np.linalg.eigvalsh((a + a.T) / 2), lam, atol=1e-12 * 10.0)


def _evd_values(A, n, b):
    import torch
    from paper_2511_16174_b200 import _lib
    L = _lib.load()
    lam = torch.empty(n, dtype=torch.float64, device="cuda")
    ws = torch.empty(L.pevd_syevd_workspace_bytes(n, b, 0, 0), dtype=torch.uint8, device="cuda")
    P = ctypes.c_void_p
    rc = L.pevd_syevd_device(n, b, P(A.data_ptr()), n, P(lam.data_ptr()), None, n, 0, 0,
                             P(ws.data_ptr()), ws.numel(),
                             P(torch.cuda.current_stream().cuda_stream), None)
    _lib.check(rc, "pevd_syevd_device")
    return lam.cpu().numpy()


@pytest.mark.parametrize("kind,n", [("Normal", 16384), ("Cluster0", 16384), ("Geometric", 8192)])
def test_planted_values_only(kind, n):
    """Config c3 (eigenvalues only, n = 16384): bisection on the device, no eigenvector merges."""
    from paper_2511_16174_b200 import matgen
    spec = matgen.SpectrumSpec(kind, n, seed=n + 11)
    A, lam_true = matgen.generate(spec)
    lam = _evd_values(A, n, 32)
    err = float(np.abs(lam - lam_true).max())
    assert err <= 10 * n * EPS * float(np.abs(lam_true).max()), f"{kind}: |dlam| {err:.3e}"
    assert np.all(np.diff(lam) >= 0)


def test_dc_standalone_65536_cluster0():
    """Config c5's solver at its own size on one GPU: the planted Cluster0 matrix (one eigenvalue
    lmax, the other 65535 at lmax / cond) is reduced to a tridiagonal T (SBR + chase), then the
    divide and conquer runs on T alone (near-total deflation).  Checked: the planted
    eigenvalues, and ||T Q - Q Lam||_F / (n ||T||_F), ||Q^T Q - I||_F / n on the device."""
    import torch
    from paper_2511_16174_b200 import _lib, matgen
    L = _lib.load()
    P = ctypes.c_void_p
    n, b = 65536, 32
    s = P(torch.cuda.current_stream().cuda_stream)
    spec = matgen.SpectrumSpec("Cluster0", n, seed=5)
    A, lam_true = matgen.generate(spec)
    bands = torch.empty((b + 1) * n, dtype=torch.float64, device="cuda")
    ws = torch.empty(L.pevd_sbr_workspace_bytes(n, b), dtype=torch.uint8, device="cuda")
    _lib.check(L.pevd_sbr(n, b, P(A.data_ptr()), n, P(bands.data_ptr()), None, P(ws.data_ptr()),
                          s), "sbr")
    del A, ws
    torch.cuda.empty_cache()
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    e = torch.empty(n, dtype=torch.float64, device="cuda")
    ws = torch.empty(L.pevd_bc_workspace_bytes(n, b), dtype=torch.uint8, device="cuda")
    _lib.check(L.pevd_bc(n, b, P(bands.data_ptr()), P(d.data_ptr()), P(e.data_ptr()), None, None,
                         32, P(ws.data_ptr()), s), "bc")
    del ws, bands
    d0, e0 = d.clone(), e[: n - 1].clone()
    Q = torch.empty((n, n), dtype=torch.float64, device="cuda")
    ws = torch.empty(L.pevd_stedc_workspace_bytes(n), dtype=torch.uint8, device="cuda")
    _lib.check(L.pevd_stedc(n, P(d.data_ptr()), P(e.data_ptr()), P(Q.data_ptr()), n,
                            P(ws.data_ptr()), s), "stedc")
    del ws
    torch.cuda.empty_cache()
    lam = d.cpu().numpy()
    err = float(np.abs(lam - lam_true).max())
    assert err <= 10 * n * EPS * float(np.abs(lam_true).max()), f"|dlam| {err:.3e}"
    # T Q - Q Lam, row block by row block (Q column-major: tensor row j = column j of Q)
    tn = float(torch.sqrt(torch.sum(d0 * d0) + 2 * torch.sum(e0 * e0)))
    res2, orth2 = 0.0, 0.0
    blk = 4096
    for j0 in range(0, n, blk):
        Qb = Q[j0:j0 + blk]                                  # columns j0.. of Q: (cols, n)
        TQ = Qb * d0[None, :]
        TQ[:, :-1] += Qb[:, 1:] * e0[None, :]
        TQ[:, 1:] += Qb[:, :-1] * e0[None, :]
        R = TQ - Qb * d[j0:j0 + blk, None]
        res2 += float(torch.sum(R * R))
        G = Qb @ Q.t()                                       # (Q^T Q)[j0.., :]
        G[:, j0:j0 + blk].diagonal().sub_(1.0)
        orth2 += float(torch.sum(G * G))
    res, orth = res2 ** 0.5 / (n * tn), orth2 ** 0.5 / n
    assert res <= 1e-12 and orth <= 1e-12, f"residual {res:.2e}, ortho {orth:.2e}"
