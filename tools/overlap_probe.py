"""Would the divide and conquer of the tridiagonal's left half overlap the second half of the
bulge chase?  Times the n = 49152 chase alone, a half-size (n/2) divide and conquer alone, and
both launched together on two streams (the D&C on a second stream as soon as the chase is
running).  Decision input for DESIGN.md section 7, not a product path.

    python tools/overlap_probe.py 49152
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_16174_b200 import _lib  # noqa: E402

P = ctypes.c_void_p
L = _lib.load()


def ptr(t):
    return P(t.data_ptr())


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 49152
    b = 32
    h = n // 2
    bands = torch.randn((b + 1) * n, dtype=torch.float64, device="cuda")
    nref = L.pevd_bc_num_reflectors(n, b)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    e = torch.empty(n, dtype=torch.float64, device="cuda")
    tau = torch.empty(nref, dtype=torch.float64, device="cuda")
    V = torch.empty(nref * b, dtype=torch.float64, device="cuda")
    wsb = torch.empty(L.pevd_bc_workspace_bytes(n, b), dtype=torch.uint8, device="cuda")
    # the half-size tridiagonal of a GOE matrix (SBR + chase: little deflation, as in the EVD)
    dh0 = torch.empty(h, dtype=torch.float64, device="cuda")
    eh = torch.empty(h, dtype=torch.float64, device="cuda")
    A = torch.randn((h, h), dtype=torch.float64, device="cuda")
    A = (A + A.t()) / 2
    bh = torch.empty((b + 1) * h, dtype=torch.float64, device="cuda")
    ws = torch.empty(L.pevd_sbr_workspace_bytes(h, b), dtype=torch.uint8, device="cuda")
    _lib.check(L.pevd_sbr(h, b, ptr(A), h, ptr(bh), None, ptr(ws), None), "sbr")
    del A, ws
    ws = torch.empty(L.pevd_bc_workspace_bytes(h, b), dtype=torch.uint8, device="cuda")
    _lib.check(L.pevd_bc(h, b, ptr(bh), ptr(dh0), ptr(eh), None, None, 32, ptr(ws), None), "bc")
    torch.cuda.synchronize()
    del ws, bh
    dh = torch.empty_like(dh0)
    Q = torch.empty((h, h), dtype=torch.float64, device="cuda")
    wsd = torch.empty(L.pevd_stedc_workspace_bytes(h), dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def chase(s):
        _lib.check(L.pevd_bc(n, b, ptr(bands), ptr(d), ptr(e), ptr(tau), ptr(V), b, ptr(wsb),
                             P(s.cuda_stream)), "bc")

    def dc(s):
        with torch.cuda.stream(s):
            dh.copy_(dh0)
        _lib.check(L.pevd_stedc(h, ptr(dh), ptr(eh), ptr(Q), h, ptr(wsd), P(s.cuda_stream)),
                   "stedc")

    def timed(fn):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s1)
        s2.wait_event(e0)
        fn()
        j = torch.cuda.Event()
        j.record(s2)
        s1.wait_event(j)
        e1.record(s1)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    out = {"n": n, "dc_n": h}
    for rep in range(2):
        out["chase_ms"] = timed(lambda: chase(s1))
        out["dc_ms"] = timed(lambda: dc(s2))
        out["both_ms"] = timed(lambda: (chase(s1), dc(s2)))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
