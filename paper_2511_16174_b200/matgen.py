"""Planted-spectrum test matrices, generated on the device.

The reference builds A = V diag(lam) V^T on the host with a Haar V from a dense QR
(matgen.py:88-126): O(n^3) host work and a 19-34 GB host->device copy at the headline sizes.
Here the spectrum is the same (`eigen_spectrum` restates matgen.py:52-84, including the Philox
SeedSequence streams of the Normal/Uniform families, and is pinned against the reference's
golden spectra), but the basis is a product of k dense Householder reflectors,

    V = H_1 H_2 ... H_k = I - Y T Y^T,     H_i = I - tau_i y_i y_i^T,  tau_i = 2 / ||y_i||^2,

drawn on the device from a seeded generator, and A = V D V^T is assembled with the FP64 DMMA
GEMM of libpevd.so as one symmetric rank-2k correction of D (O(k n^2) flops):

    W = Y T,  M = D Y,  S = Y^T M,  Z = M - W S / 2,  A = D - (W Z^T + Z W^T).

The planted eigenvalues are exact up to the rounding of that assembly, so an EVD of any size can
be checked against known eigenvalues, and `accuracy` measures the north star's residual and
orthogonality blockwise on the device (the check itself is verification, not the product path).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

KINDS = ("Cluster0", "Cluster1", "Geometric", "Arithmetic", "Normal", "Uniform")
_CANON = {k.lower(): k for k in KINDS}


def canonical_kind(name: str) -> str:
    """Case-insensitive family lookup (matgen.py:24-29)."""
    try:
        return _CANON[name.lower()]
    except KeyError:
        raise ValueError(f"unknown spectrum kind {name!r}; choose from {KINDS}") from None


@dataclass
class SpectrumSpec:
    """Spectrum family and its parameters (matgen.py:32-45)."""

    kind: str
    n: int
    cond: float = 1e8
    lambda_max: float = 1e6
    seed: int = 0

    def __post_init__(self):
        self.kind = canonical_kind(self.kind)
        if self.cond < 1.0:
            raise ValueError("cond must be >= 1")
        if self.lambda_max <= 0.0:
            raise ValueError("lambda_max must be positive")


def _philox(entropy):
    return np.random.Generator(np.random.Philox(entropy))


def eigen_spectrum(spec: SpectrumSpec) -> np.ndarray:
    """n eigenvalues of the family, ascending (matgen.py:52-84)."""
    n = spec.n
    if n < 2:
        raise ValueError("spectrum needs n >= 2")
    top, cond = spec.lambda_max, spec.cond
    i = np.arange(n, dtype=np.float64)
    if spec.kind == "Cluster0":      # one at lambda_max, the rest at lambda_max / cond
        lam = np.full(n, top / cond)
        lam[0] = top
    elif spec.kind == "Cluster1":    # n - 1 at lambda_max, one at lambda_max / cond
        lam = np.full(n, top)
        lam[-1] = top / cond
    elif spec.kind == "Geometric":
        lam = top * cond ** (-i / (n - 1))
    elif spec.kind == "Arithmetic":
        lam = top * (1.0 - (1.0 - 1.0 / cond) * i / (n - 1))
    else:                            # Normal / Uniform: first child of the seed sequence
        rng = _philox(np.random.SeedSequence(spec.seed).spawn(2)[0])
        lam = rng.standard_normal(n) if spec.kind == "Normal" else rng.uniform(-1.0, 1.0, n)
    return np.sort(lam)


def householder_t(gram: np.ndarray) -> np.ndarray:
    """T (k x k upper) of H_1 ... H_k = I - Y T Y^T from G = Y^T Y (LAPACK larft 'F', columnwise):
    T_ii = tau_i = 2 / G_ii, T[:i, i] = -tau_i T[:i, :i] G[:i, i]."""
    k = gram.shape[0]
    t = np.zeros((k, k))
    for i in range(k):
        tau = 2.0 / gram[i, i]
        t[i, i] = tau
        if i:
            t[:i, i] = -tau * (t[:i, :i] @ gram[:i, i])
    return t


class _Dev:
    """Column-major device matrices over the C-ABI GEMM (a col-major rows x cols matrix is a torch
    tensor of shape (cols, rows))."""

    def __init__(self):
        self.torch = _lib.require_cuda()
        self.L = _lib.load()
        self.ws = self.torch.empty(64 << 20, dtype=self.torch.uint8, device="cuda")

    def gemm(self, A, B, C, alpha=1.0, beta=0.0, ta=False, tb=False):
        m = A.shape[0] if ta else A.shape[1]
        k = A.shape[1] if ta else A.shape[0]
        n = B.shape[1] if tb else B.shape[0]
        P = ctypes.c_void_p
        s = P(self.torch.cuda.current_stream().cuda_stream)
        rc = self.L.pevd_dgemm(int(ta), int(tb), m, n, k, alpha, P(A.data_ptr()), A.stride(0),
                               P(B.data_ptr()), B.stride(0), beta, P(C.data_ptr()), C.stride(0),
                               P(self.ws.data_ptr()), self.ws.numel(), s)
        _lib.check(rc, "dgemm")


def planted(lam, k: int = 64, seed: int = 0, out=None):
    """A = V diag(lam) V^T on the current CUDA device, column-major (a torch tensor of shape
    (n, n) whose transpose is A; A is symmetric, so the tensor is A up to rounding).
    V is the product of k dense Householder reflectors drawn from `seed`."""
    d = _Dev()
    torch = d.torch
    lam_h = np.asarray(lam, dtype=np.float64)
    n = lam_h.shape[0]
    k = max(1, min(k, n))
    g = torch.Generator(device="cuda")
    g.manual_seed(int(seed))
    Y = torch.randn((k, n), dtype=torch.float64, device="cuda", generator=g)  # col-major n x k
    G = torch.empty((k, k), dtype=torch.float64, device="cuda")
    d.gemm(Y, Y, G, ta=True)                                                  # G = Y^T Y
    T = torch.from_numpy(np.ascontiguousarray(householder_t(G.cpu().numpy().T).T)).cuda()
    W = torch.empty_like(Y)
    d.gemm(Y, T, W)                                                           # W = Y T
    lam_d = torch.from_numpy(lam_h).cuda()
    M = Y * lam_d                                                             # D Y (row scaling)
    S = torch.empty((k, k), dtype=torch.float64, device="cuda")
    d.gemm(Y, M, S, ta=True)                                                  # S = Y^T D Y
    d.gemm(W, S, M, alpha=-0.5, beta=1.0)                                     # Z = M - W S / 2
    A = out if out is not None else torch.empty((n, n), dtype=torch.float64, device="cuda")
    A.zero_()
    A.diagonal().copy_(lam_d)
    d.gemm(W, M, A, alpha=-1.0, beta=1.0, tb=True)                            # A -= W Z^T
    d.gemm(M, W, A, alpha=-1.0, beta=1.0, tb=True)                            # A -= Z W^T
    return A


def generate(spec: SpectrumSpec, k: int = 64, out=None):
    """(device A, planted spectrum) for a SpectrumSpec; basis seed = spec.seed."""
    lam = eigen_spectrum(spec)
    return planted(lam, k=k, seed=spec.seed, out=out), lam


def accuracy(A, lam, Q, block: int = 4096):
    """North-star accuracy on the device, blockwise over the columns of Q (n x block scratch):
    residual ||A Q - Q Lam||_F / (n ||A||_F) and orthogonality ||Q^T Q - I||_F / n.
    A, Q: column-major device tensors (shape (n, n)); lam: device or host vector."""
    d = _Dev()
    torch = d.torch
    n = Q.shape[0]
    lam_d = torch.as_tensor(np.asarray(lam.cpu() if hasattr(lam, "cpu") else lam),
                            dtype=torch.float64).cuda()
    res2, orth2 = 0.0, 0.0
    R = torch.empty((min(block, n), n), dtype=torch.float64, device="cuda")
    for j0 in range(0, n, block):
        j1 = min(n, j0 + block)
        Qb = Q[j0:j1]                              # columns j0..j1 of Q (col-major view)
        Rb = R[: j1 - j0]
        Rb.copy_(Qb * lam_d[j0:j1, None])          # Q_blk Lam_blk
        d.gemm(A, Qb, Rb, alpha=1.0, beta=-1.0)    # A Q_blk - Q_blk Lam_blk
        res2 += float(torch.sum(Rb * Rb))
        d.gemm(Q, Qb, Rb, ta=True)                 # Q^T Q_blk
        Rb[:, j0:j1].diagonal().sub_(1.0)
        orth2 += float(torch.sum(Rb * Rb))
    anorm = float(torch.linalg.norm(A))
    return (res2 ** 0.5) / (n * anorm), (orth2 ** 0.5) / n


# ---------------------------------------------------------------- host generator (CLI `gen`)
def random_orthogonal(n: int, seed) -> np.ndarray:
    """Haar orthogonal matrix from a Philox stream (matgen.py:87-103): QR of a Gaussian matrix
    with the signs of R's diagonal moved into Q (zero counts as +)."""
    if n < 1:
        raise ValueError("n >= 1 required")
    ss = seed if isinstance(seed, np.random.SeedSequence) else np.random.SeedSequence(seed)
    g = _philox(ss).standard_normal((n, n))
    q, r = np.linalg.qr(g)
    return np.asfortranarray(q * np.where(np.diag(r) < 0.0, -1.0, 1.0))


def generate_host(spec: SpectrumSpec):
    """(A, lam) exactly as the reference CLI's `gen` builds them (matgen.py:106-126): the basis
    from the second child of the seed sequence, A = (V diag(lam) V^T + its transpose) / 2.
    O(n^3) host work: the reference-compatible path for files; `generate` is the device one."""
    lam = eigen_spectrum(spec)
    v = random_orthogonal(spec.n, np.random.SeedSequence(spec.seed).spawn(2)[1])
    a = (v * lam) @ v.T
    return np.asfortranarray((a + a.T) / 2.0), lam
