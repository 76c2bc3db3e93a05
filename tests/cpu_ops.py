"""CPU implementation of the distributed driver's compute interface -- TEST INFRASTRUCTURE.

Lets tests run paper_2511_16174_b200.distributed.run_distributed under the gloo backend on a
machine without a GPU: the protocol (partition, panel gathers, broadcasts, all-gathers, row
blocks, ledger) is the product's; the arithmetic here is the oracle's.
"""
import numpy as np
import torch

from oracle import oracle as orc


class CpuOps:
    device = torch.device("cpu")

    def from_host(self, a):
        return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64).T).copy())

    def to_host(self, t):
        return np.asfortranarray(t.detach().numpy().T)

    def zeros(self, rows, cols):
        return torch.zeros((cols, rows), dtype=torch.float64)

    def gemm(self, A, B, C, alpha=1.0, beta=0.0, ta=False, tb=False):
        Am = A.T if not ta else A        # column-major view (cols, rows) -> matrix via .T
        Bm = B.T if not tb else B
        res = alpha * (Am @ Bm)
        if beta != 0.0:
            res = res + beta * C.T
        C.T.copy_(res)

    def panel_qr(self, P):
        p = np.asfortranarray(P.numpy().T.copy())     # m x pw
        W, Y = orc.panel_qr(p)
        k = Y.shape[1]
        T = np.triu(np.linalg.lstsq(Y, W, rcond=None)[0])
        R = np.triu(p[:k, :])
        return self.from_host(R), self.from_host(Y), self.from_host(T)

    def bc(self, bands):
        b = np.ascontiguousarray(bands.numpy())
        d, e, refl = orc.bc_reduce(b)
        return d, e, refl, None

    def stedc(self, d, e, cols=None):
        lam, q = orc.tridiag_eig(np.asarray(d), np.asarray(e), want_vectors=True)
        if cols is not None:  # mimic the device: only the requested columns are formed
            q2 = np.zeros_like(q)
            q2[:, cols[0]:cols[1]] = q[:, cols[0]:cols[1]]
            q = q2
        return lam, self.from_host(q)

    def bc_back_left(self, n, b, refl, _, X):
        x = self.to_host(X)                              # n x cols
        return self.from_host(orc.bc_back_apply(refl, x, "conventional"))

    def bc_back_right(self, n, b, refl, _, X):
        x = self.to_host(X)                              # rows x n
        out = orc.bc_back_apply(refl, x.T, "reordered").T
        return self.from_host(out)
