"""BC-Back kernel check + timing: apply the bulge reflectors of
a random band to a random X through pevd_bc_back_left (conventional, on the transpose) and
pevd_bc_back_right, compare with the CPU oracle at small n, time at large n.

    python tools/bcb_check.py 2048 32768
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_16174_b200 import _lib, device  # noqa: E402

P = ctypes.c_void_p
L = _lib.load()


def refl(n, b, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    bands = torch.randn((b + 1) * n, dtype=torch.float64, device="cuda", generator=g)
    nref = L.pevd_bc_num_reflectors(n, b)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    e = torch.empty(n, dtype=torch.float64, device="cuda")
    tau = torch.empty(nref, dtype=torch.float64, device="cuda")
    V = torch.empty(nref * 32, dtype=torch.float64, device="cuda")
    ws = torch.empty(L.pevd_bc_workspace_bytes(n, b), dtype=torch.uint8, device="cuda")
    _lib.check(L.pevd_bc(n, b, P(bands.data_ptr()), P(d.data_ptr()), P(e.data_ptr()),
                         P(tau.data_ptr()), P(V.data_ptr()), 32, P(ws.data_ptr()),
                         P(torch.cuda.current_stream().cuda_stream)), "bc")
    return tau, V


def apply(fn, n, tau, V, X):
    ws = torch.empty(L.pevd_bc_back_workspace_bytes(n, n, 32), dtype=torch.uint8, device="cuda")
    _lib.check(fn(n, 32, P(tau.data_ptr()), P(V.data_ptr()), 32, P(X.data_ptr()), n, n,
                  P(ws.data_ptr()), P(torch.cuda.current_stream().cuda_stream)), "bc_back")


def main():
    out = {}
    n = int(sys.argv[1])
    tau, V = refl(n, 32, 1)
    X0 = torch.randn((n, n), dtype=torch.float64, device="cuda")
    # oracle
    from oracle import oracle as orc
    r = device.slots_to_reference(n, 32, tau.cpu().numpy(), V.cpu().numpy().reshape(-1, 32))
    x0 = X0.cpu().numpy().T.copy()  # column-major (n x n): the tensor's transpose
    for name, fn, direction in (("left", L.pevd_bc_back_left, "conventional"),
                                ("right", L.pevd_bc_back_right, "reordered")):
        X = X0.clone()
        apply(fn, n, tau, V, X)
        got = X.cpu().numpy().T
        if direction == "conventional":
            want = orc.bc_back_apply(r, x0, "conventional")
        else:  # X <- X Q_b on the rows: (Q_b^T X^T)^T
            want = orc.bc_back_apply(r, x0.T.copy(), "reordered").T
        out[name + "_maxdiff"] = float(np.abs(got - want).max())
    for nn in (int(x) for x in sys.argv[2:]):
        tau, V = refl(nn, 32, 2)
        X = torch.randn((nn, nn), dtype=torch.float64, device="cuda")
        for name, fn in (("left", L.pevd_bc_back_left), ("right", L.pevd_bc_back_right)):
            apply(fn, nn, tau, V, X)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            apply(fn, nn, tau, V, X)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            out[f"{name}_{nn}_ms"] = round(ms, 1)
            out[f"{name}_{nn}_tflops_blas2"] = round(2 * nn ** 3 / ms / 1e9, 2)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
