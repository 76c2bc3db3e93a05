"""Where the end-to-end overhead of pevd_syevd (HOST buffers) goes at n = 49152: device
allocation (cudaMalloc / cudaFree of A, Q and the workspace), the lower-trapezoid upload from
pinned memory, and the whole call against its own device stage span.

    python tools/hostio_probe.py 49152
"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_16174_b200 import _lib  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 49152
    L = _lib.load()
    rt = ctypes.CDLL("libcudart.so.12")
    rt.cudaMalloc.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t]
    rt.cudaFree.argtypes = [ctypes.c_void_p]
    rt.cudaDeviceSynchronize.argtypes = []
    torch.cuda.init()
    torch.empty(1, device="cuda")  # context up before anything is timed
    wsb = L.pevd_syevd_workspace_bytes(n, 32, 1, 2)
    out = {"n": n, "workspace_gb": round(wsb / 1e9, 2)}
    ptrs = []
    t = time.perf_counter()
    for nbytes in (n * n * 8, n * n * 8, wsb):
        p = ctypes.c_void_p()
        assert rt.cudaMalloc(ctypes.byref(p), nbytes) == 0
        ptrs.append(p)
    rt.cudaDeviceSynchronize()
    out["malloc_s"] = round(time.perf_counter() - t, 4)
    t = time.perf_counter()
    for p in ptrs:
        rt.cudaFree(p)
    rt.cudaDeviceSynchronize()
    out["free_s"] = round(time.perf_counter() - t, 4)

    a = torch.randn((n, n), dtype=torch.float64, device="cuda")
    a_host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    a_host.copy_(a)
    d = torch.empty_like(a)
    torch.cuda.synchronize()
    t = time.perf_counter()
    d.copy_(a_host, non_blocking=True)
    torch.cuda.synchronize()
    out["full_h2d_pinned_s"] = round(time.perf_counter() - t, 4)
    t = time.perf_counter()
    a_host.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    out["full_d2h_pinned_s"] = round(time.perf_counter() - t, 4)
    del a, d
    torch.cuda.empty_cache()

    a = torch.randn((n, n), dtype=torch.float64, device="cuda")
    a.add_(a.t().clone())
    a_host.copy_(a)
    del a
    torch.cuda.empty_cache()
    q_host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    lam_host = torch.empty(n, dtype=torch.float64, pin_memory=True)
    P = ctypes.c_void_p
    for rep in range(2):
        st = _lib.PevdStats()
        t = time.perf_counter()
        rc = L.pevd_syevd(n, 32, P(a_host.data_ptr()), n, P(lam_host.data_ptr()),
                          P(q_host.data_ptr()), n, 1, 2, ctypes.byref(st))
        wall = time.perf_counter() - t
        _lib.check(rc, "pevd_syevd")
        out[f"call{rep}"] = {"wall_s": round(wall, 3), "device_span_s": round(st.total_ms / 1e3, 3),
                             "overhead_s": round(wall - st.total_ms / 1e3, 3),
                             "sbr_back_s": round((st.sbr_back_ms[1] - st.sbr_back_ms[0]) / 1e3, 3),
                             "bc_back_s": round((st.bc_back_ms[1] - st.bc_back_ms[0]) / 1e3, 3)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
