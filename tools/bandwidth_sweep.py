"""Stage times of the single-GPU EVD (conventional order, eigenvectors) across the band-width
parameter b at one n: what the wider bands (b > 32: the wide chase kernel, the 64-column panel
QR, the DMMA BC-Back for multiples of 8) and the generic BC-Back (other b) cost.

    python tools/bandwidth_sweep.py 16384 16 24 32 40 48 64 36
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_16174_b200 import _lib  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    bs = [int(x) for x in sys.argv[2:]] or [16, 24, 32, 40, 48, 64]
    L = _lib.load()
    P = ctypes.c_void_p
    g = torch.Generator(device="cuda")
    g.manual_seed(n)
    a0 = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    a0.add_(a0.t().clone())
    for b in bs:
        oc = _lib.ORDER_CODES["conventional"]
        ws = torch.empty(L.pevd_syevd_workspace_bytes(n, b, 1, oc), dtype=torch.uint8, device="cuda")
        q = torch.empty((n, n), dtype=torch.float64, device="cuda")
        lam = torch.empty(n, dtype=torch.float64, device="cuda")
        for rep in range(2):
            a = a0.clone()
            st = _lib.PevdStats()
            rc = L.pevd_syevd_device(n, b, P(a.data_ptr()), n, P(lam.data_ptr()), P(q.data_ptr()), n,
                                     1, oc, P(ws.data_ptr()), ws.numel(),
                                     P(torch.cuda.current_stream().cuda_stream), ctypes.byref(st))
            _lib.check(rc, "pevd_syevd_device")
        span = lambda x: round((x[1] - x[0]) / 1e3, 3)  # noqa: E731
        print(json.dumps({"n": n, "b": b, "total_s": round(st.total_ms / 1e3, 3),
                          "tflops_4n3": round(4 * n ** 3 / (st.total_ms * 1e-3) / 1e12, 2),
                          "sbr": span(st.sbr_ms), "bc": span(st.bc_ms), "solver": span(st.solver_ms),
                          "bc_back": span(st.bc_back_ms), "sbr_back": span(st.sbr_back_ms)}),
              flush=True)
        del ws, q, a
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
