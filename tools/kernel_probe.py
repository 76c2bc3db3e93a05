"""Time individual device stages through the C ABI (CUDA events, after warm-up).

  python tools/kernel_probe.py bcback 16384        # BC-Back on n x n rows
  python tools/kernel_probe.py gemm 8192 8192 8192 [ta tb]
  python tools/kernel_probe.py sbr 16384
  python tools/kernel_probe.py stedc 16384
  python tools/kernel_probe.py bc 16384
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


def stream():
    return P(torch.cuda.current_stream().cuda_stream)


def timed(fn, reps=3, warm=1):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts), ts


def rand_band(n, b, seed=0):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return torch.randn((b + 1) * n, dtype=torch.float64, device="cuda", generator=g)


def reflectors(n, b):
    bands = rand_band(n, b)
    nref = L.pevd_bc_num_reflectors(n, b)
    vld = (b + 7) // 8 * 8
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    e = torch.empty(n, dtype=torch.float64, device="cuda")
    tau = torch.empty(nref, dtype=torch.float64, device="cuda")
    V = torch.empty(nref * vld, dtype=torch.float64, device="cuda")
    ws = torch.empty(L.pevd_bc_workspace_bytes(n, b), dtype=torch.uint8, device="cuda")
    ms, _ = timed(lambda: _lib.check(L.pevd_bc(n, b, ptr(bands), ptr(d), ptr(e), ptr(tau), ptr(V),
                                               vld, ptr(ws), stream()), "bc"), reps=1, warm=0)
    return tau, V, vld, ms


def main():
    mode = sys.argv[1]
    out = {"mode": mode}
    if mode in ("bcback", "bcbackl"):
        n = int(sys.argv[2])
        b = 32
        tau, V, vld, _ = reflectors(n, b)
        X = torch.randn((n, n), dtype=torch.float64, device="cuda")
        ws = torch.empty(L.pevd_bc_back_workspace_bytes(n, n, 32), dtype=torch.uint8, device="cuda")
        fn = L.pevd_bc_back_right if mode == "bcback" else L.pevd_bc_back_left
        ms, ts = timed(lambda: _lib.check(fn(n, b, ptr(tau), ptr(V), vld, ptr(X), n, n, ptr(ws),
                                             stream()), mode))
        nref = L.pevd_bc_num_reflectors(n, b)
        flops = 4.0 * b * nref * n
        out.update(n=n, ms=ms, ts=ts,
                   tflops=flops / ms / 1e9)
    elif mode == "bc":
        n = int(sys.argv[2])
        _, _, _, ms = reflectors(n, 32)
        _, _, _, ms = reflectors(n, 32)
        out.update(n=n, ms=ms, us_per_slot=ms * 1e3 / (3 * n))
    elif mode == "gemm":
        m, n, k = (int(x) for x in sys.argv[2:5])
        ta = int(sys.argv[5]) if len(sys.argv) > 5 else 0
        tb = int(sys.argv[6]) if len(sys.argv) > 6 else 0
        beta = float(sys.argv[7]) if len(sys.argv) > 7 else 0.0
        A = torch.randn(m * k, dtype=torch.float64, device="cuda")
        B = torch.randn(k * n, dtype=torch.float64, device="cuda")
        C = torch.zeros(m * n, dtype=torch.float64, device="cuda")
        ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
        lda = k if ta else m
        ldb = n if tb else k
        ms, ts = timed(lambda: _lib.check(L.pevd_dgemm(ta, tb, m, n, k, 1.0, ptr(A), lda, ptr(B), ldb,
                                                       beta, ptr(C), m, ptr(ws), ws.numel(), stream()),
                                          "gemm"), reps=5)
        out.update(m=m, n=n, k=k, ms=ms, tflops=2.0 * m * n * k / ms / 1e9)
    elif mode == "gemm_grouped":
        # pevd_dgemm vs the grouped path (D&C merges) on one shape; cmap = 1 adds a column map
        m, n, k = (int(x) for x in sys.argv[2:5])
        use_map = len(sys.argv) > 5 and sys.argv[5] == "1"
        A = torch.randn(m * k, dtype=torch.float64, device="cuda")
        B = torch.randn(k * n, dtype=torch.float64, device="cuda")
        C = torch.zeros(m * n, dtype=torch.float64, device="cuda")
        cmap = torch.arange(n, dtype=torch.int32, device="cuda") if use_map else None
        dargs = torch.empty(4096, dtype=torch.uint8, device="cuda")
        L.pevd_probe_gemm_grouped.argtypes = [ctypes.c_int64] * 3 + [P, ctypes.c_int64, P,
                                              ctypes.c_int64, P, ctypes.c_int64, P, P, P]
        msg, _ = timed(lambda: _lib.check(L.pevd_probe_gemm_grouped(
            m, n, k, ptr(A), m, ptr(B), k, ptr(C), m, ptr(cmap) if use_map else None,
            ptr(dargs), stream()), "grouped"), reps=3)
        ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
        msp, _ = timed(lambda: _lib.check(L.pevd_dgemm(0, 0, m, n, k, 1.0, ptr(A), m, ptr(B), k,
                                                       0.0, ptr(C), m, ptr(ws), ws.numel(),
                                                       stream()), "gemm"), reps=3)
        out.update(m=m, n=n, k=k, cmap=use_map, grouped_tflops=2.0 * m * n * k / msg / 1e9,
                   plain_tflops=2.0 * m * n * k / msp / 1e9)
    elif mode == "symm":
        m, n = int(sys.argv[2]), int(sys.argv[3])
        lda = int(sys.argv[4]) if len(sys.argv) > 4 else m  # the SBR passes lda = n_total
        A = torch.randn(lda * m, dtype=torch.float64, device="cuda")
        B = torch.randn(lda * n, dtype=torch.float64, device="cuda")
        C = torch.zeros(lda * n, dtype=torch.float64, device="cuda")
        ws = torch.empty(int(os.environ.get("PROBE_WS_MB", "32")) << 20, dtype=torch.uint8, device="cuda")
        ms, ts = timed(lambda: _lib.check(L.pevd_dsymm_lower(m, n, 1.0, ptr(A), lda, ptr(B), lda,
                                                             0.0, ptr(C), lda, ptr(ws),
                                                             ws.numel(), stream()), "symm"),
                       reps=5)
        out.update(m=m, n=n, lda=lda, ms=ms, tflops=2.0 * m * m * n / ms / 1e9,
                   gbs=8.0 * m * m / ms / 1e6)
    elif mode == "sbr":
        n = int(sys.argv[2])
        b = 32
        A0 = torch.randn((n, n), dtype=torch.float64, device="cuda")
        A0 = (A0 + A0.t()) / 2
        A = torch.empty_like(A0)
        bands = torch.empty((b + 1) * n, dtype=torch.float64, device="cuda")
        tall = torch.empty(((n - b) // b + 1) * b * b, dtype=torch.float64, device="cuda")
        ws = torch.empty(L.pevd_sbr_workspace_bytes(n, b), dtype=torch.uint8, device="cuda")

        def f():
            A.copy_(A0)
            _lib.check(L.pevd_sbr(n, b, ptr(A), n, ptr(bands), ptr(tall), ptr(ws), stream()), "sbr")
        ms, ts = timed(f, reps=2)
        out.update(n=n, ms=ms, tflops=4 * n ** 3 / 3 / ms / 1e9)
    elif mode in ("sbrback", "sbrform"):
        # SBR once (its Y staircase and T factors), then time SBR-Back on an n x n X
        n = int(sys.argv[2])
        b = 32
        A = torch.randn((n, n), dtype=torch.float64, device="cuda")
        A = (A + A.t()) / 2
        bands = torch.empty((b + 1) * n, dtype=torch.float64, device="cuda")
        tall = torch.empty(((n - b) // b + 1) * b * b, dtype=torch.float64, device="cuda")
        ws = torch.empty(L.pevd_sbr_workspace_bytes(n, b), dtype=torch.uint8, device="cuda")
        _lib.check(L.pevd_sbr(n, b, ptr(A), n, ptr(bands), ptr(tall), ptr(ws), stream()), "sbr")
        del ws
        X = torch.randn((n, n), dtype=torch.float64, device="cuda")
        ws = torch.empty(L.pevd_sbr_back_workspace_bytes(n, b), dtype=torch.uint8, device="cuda")
        if mode == "sbrback":
            fn = lambda: _lib.check(L.pevd_sbr_back_left(n, b, ptr(A), n, ptr(tall), ptr(X), n, n,  # noqa
                                                         ptr(ws), stream()), "sbr_back_left")
            flops = 2.0 * n ** 3
        else:
            fn = lambda: _lib.check(L.pevd_sbr_back_form(n, b, ptr(A), n, ptr(tall), ptr(X), n,  # noqa
                                                         ptr(ws), stream()), "sbr_back_form")
            flops = 4.0 * n ** 3 / 3
        ms, ts = timed(fn, reps=2)
        out.update(n=n, nbagg=os.environ.get("PEVD_NBAGG", "default"), ms=ms,
                   tflops=flops / ms / 1e9)
    elif mode == "pqr":
        # panel QR of an m x 32 panel (the SBR critical path)
        m = int(sys.argv[2])
        k = 32
        P0 = torch.randn((k, m), dtype=torch.float64, device="cuda")
        Pn = torch.empty_like(P0)
        R = torch.empty((k, k), dtype=torch.float64, device="cuda")
        Y = torch.empty((k, m), dtype=torch.float64, device="cuda")
        T = torch.empty((k, k), dtype=torch.float64, device="cuda")
        ws = torch.empty(L.pevd_panel_qr_workspace_bytes(), dtype=torch.uint8, device="cuda")

        def f():
            for _ in range(20):
                _lib.check(L.pevd_panel_qr(m, k, ptr(P0), m, ptr(R), ptr(Y), m, None, m, ptr(T),
                                           ptr(ws), stream()), "pqr")
        ms, ts = timed(f, reps=3)
        out.update(m=m, us_per_panel=ms * 1e3 / 20)
    elif mode in ("stedc", "stedc_goe"):
        n = int(sys.argv[2])
        d0 = torch.randn(n, dtype=torch.float64, device="cuda")
        e = torch.randn(n, dtype=torch.float64, device="cuda")
        if mode == "stedc_goe":  # the tridiagonal of a GOE matrix (SBR + chase): little deflation
            b = 32
            A = torch.randn((n, n), dtype=torch.float64, device="cuda")
            A = (A + A.t()) / 2
            bands = torch.empty((b + 1) * n, dtype=torch.float64, device="cuda")
            ws = torch.empty(L.pevd_sbr_workspace_bytes(n, b), dtype=torch.uint8, device="cuda")
            _lib.check(L.pevd_sbr(n, b, ptr(A), n, ptr(bands), None, ptr(ws), stream()), "sbr")
            del A, ws
            ws = torch.empty(L.pevd_bc_workspace_bytes(n, b), dtype=torch.uint8, device="cuda")
            _lib.check(L.pevd_bc(n, b, ptr(bands), ptr(d0), ptr(e), None, None, 32, ptr(ws),
                                 stream()), "bc")
            del ws
        d = torch.empty_like(d0)
        Q = torch.empty((n, n), dtype=torch.float64, device="cuda")
        ws = torch.empty(L.pevd_stedc_workspace_bytes(n), dtype=torch.uint8, device="cuda")

        def f():
            d.copy_(d0)
            _lib.check(L.pevd_stedc(n, ptr(d), ptr(e), ptr(Q), n, ptr(ws), stream()), "stedc")
        ms, ts = timed(f, reps=2)
        out.update(n=n, ms=ms)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
