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

    def bc_partition(self, tail, b, c0, pend, n):
        """The relayed chase of one partition (bulge.py:348-385) on the oracle's dense chase:
        sweeps [c0, pend) on the band tail [c0, n).  Returns d, e (final for the partition's
        columns), the band tail beyond pend and the reflectors (global indices)."""
        bands = np.ascontiguousarray(tail.numpy() if hasattr(tail, "numpy") else tail)
        m = n - c0
        full = np.zeros((2 * b + 1, m))
        full[: bands.shape[0]] = bands[:, :m]
        s = np.ascontiguousarray(orc.band_to_dense(full))
        stride = orc.pad8(b)
        cap = max(orc.step_capacity(n, b, c0, pend), 1)
        ia = np.zeros(cap, np.int64); ja = np.zeros(cap, np.int64)
        ra = np.zeros(cap, np.int64); la = np.zeros(cap, np.int64)
        ta = np.zeros(cap); va = np.zeros((cap, stride))
        import ctypes
        macs = ctypes.c_int64(0)
        P = orc._p
        cnt = orc.lib().orc_chase(P(s), m, c0, n, b, c0, pend, P(ia, orc._i64p), P(ja, orc._i64p),
                                  P(ra, orc._i64p), P(la, orc._i64p), P(ta), P(va), stride,
                                  ctypes.byref(macs))
        refl = dict(i=ia[:cnt], j=ja[:cnt], row0=ra[:cnt], len=la[:cnt], tau=ta[:cnt],
                    v=va[:cnt])
        out = np.zeros((2 * b + 1, m))
        for dd in range(2 * b + 1):
            out[dd, : m - dd] = np.diag(s, -dd)
        last = pend >= n
        npiv = pend - c0
        d = out[0, :m].copy() if last else out[0, :npiv].copy()
        e = out[1, : m - 1].copy() if last else out[1, :npiv].copy()
        mr = n - pend
        bwo = min(2 * b, max(mr - 1, 0))
        tailo = torch.from_numpy(np.ascontiguousarray(out[: bwo + 1, npiv:])) if not last else None
        return {"d": d, "e": e, "tail": tailo, "refl": refl}

    def merge_reflectors(self, sets):
        """All partitions' reflectors in the canonical (j outer, i inner) order (bulge.py:126-141)."""
        keys = ("i", "j", "row0", "len", "tau", "v")
        cat = {k: np.concatenate([np.asarray(s_[k]) for s_ in sets]) for k in keys}
        perm = np.lexsort((cat["i"], cat["j"]))
        return {k: cat[k][perm] for k in keys}

    def stedc(self, d, e, cols=None):
        lam, q = orc.tridiag_eig(np.asarray(d, dtype=np.float64), np.asarray(e, dtype=np.float64),
                                 want_vectors=True)
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
