"""Bitwise fingerprint of the bulge chase's outputs (d, e, tau, V) on fixed random bands, for
comparing the lag-2 and lag-3 wavefront kernels (PEVD_CHASE_LAG=2 / 3): both must perform
exactly the sequential chase's operations, so their outputs must be identical bit for bit.

    PEVD_CHASE_LAG=3 python tools/chase_lag_check.py > a;  python tools/chase_lag_check.py > b
"""
import ctypes
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_16174_b200 import _lib  # noqa: E402

P = ctypes.c_void_p
L = _lib.load()


def run(n, b, reps):
    g = torch.Generator(device="cuda")
    g.manual_seed(n * 100 + b)
    bands = torch.randn((b + 1) * n, dtype=torch.float64, device="cuda", generator=g)
    nref = L.pevd_bc_num_reflectors(n, b)
    vld = (b + 7) // 8 * 8
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    e = torch.empty(n, dtype=torch.float64, device="cuda")
    tau = torch.empty(max(nref, 1), dtype=torch.float64, device="cuda")
    V = torch.empty(max(nref, 1) * vld, dtype=torch.float64, device="cuda")
    ws = torch.empty(L.pevd_bc_workspace_bytes(n, b), dtype=torch.uint8, device="cuda")
    digests, ms = set(), []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.check(L.pevd_bc(n, b, P(bands.data_ptr()), P(d.data_ptr()), P(e.data_ptr()),
                             P(tau.data_ptr()), P(V.data_ptr()), vld, P(ws.data_ptr()), None), "bc")
        torch.cuda.synchronize()
        ms.append((time.perf_counter() - t0) * 1e3)
        h = hashlib.sha256()
        for t in (d, e, tau, V):
            h.update(t.cpu().numpy().tobytes())
        digests.add(h.hexdigest()[:16])
    out = os.environ.get("CHASE_SAVE")
    if out and n <= 20001:
        import numpy as np
        np.savez(f"{out}_{n}_{b}.npz", d=d.cpu().numpy(), e=e.cpu().numpy(),
                 tau=tau.cpu().numpy(), V=V.cpu().numpy())
    return {"n": n, "b": b, "digests": sorted(digests), "ms": round(min(ms), 2)}


def compare(a, b):
    """max |difference| per output between two CHASE_SAVE runs, and the first differing slot"""
    import glob
    import numpy as np
    for fa in sorted(glob.glob(f"{a}_*.npz")):
        fb = fa.replace(a, b, 1)
        A, B = np.load(fa), np.load(fb)
        row = {"case": fa}
        for k in ("d", "e", "tau", "V"):
            diff = np.abs(A[k] - B[k])
            row[k] = float(diff.max()) if diff.size else 0.0
            if k == "tau" and diff.max() > 0:
                row["first_tau_slot"] = int(np.argmax(diff > 0))
        print(json.dumps(row))


def main():
    if len(sys.argv) == 4 and sys.argv[1] == "compare":
        return compare(sys.argv[2], sys.argv[3])
    cases = [(40, 8), (300, 16), (1000, 32), (1001, 24), (4097, 32), (16384, 32), (20001, 8),
             (49152, 32)]
    for n, b in cases:
        print(json.dumps(run(n, b, 3 if n <= 20001 else 2)), flush=True)


if __name__ == "__main__":
    main()
