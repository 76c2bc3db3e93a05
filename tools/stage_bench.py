"""Stage timing of the single-GPU EVD at several n (device-resident input, CUDA-event stages).

python tools/stage_bench.py 8192 16384 [--check] [--order pipelined]
Prints one JSON line per n with per-stage [start, end] ms and, with --check, the residual and
orthogonality (computed with torch on the device; verification only).
"""
import argparse
import ctypes
import json
import time

import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2511_16174_b200 import _lib


def sym_on_device(n, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    a = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    a.add_(a.t().clone())
    a.mul_(0.5)
    return a


def run(n, b, order, check, reps):
    L = _lib.load()
    oc = _lib.ORDER_CODES[order]
    a0 = sym_on_device(n, n)
    ws = torch.empty(L.pevd_syevd_workspace_bytes(n, b, 1, oc), dtype=torch.uint8, device="cuda")
    lam = torch.empty(n, dtype=torch.float64, device="cuda")
    q = torch.empty((n, n), dtype=torch.float64, device="cuda")
    a = torch.empty_like(a0)
    out = []
    for r in range(reps):
        a.copy_(a0)
        st = _lib.PevdStats()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc = L.pevd_syevd_device(n, b, ctypes.c_void_p(a.data_ptr()), n,
                                 ctypes.c_void_p(lam.data_ptr()), ctypes.c_void_p(q.data_ptr()), n,
                                 1, oc, ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream),
                                 ctypes.byref(st))
        wall = time.perf_counter() - t0
        _lib.check(rc, "syevd")
        rec = dict(n=n, b=b, order=order, rep=r, wall_s=round(wall, 4),
                   tflops_4n3=round(4 * n ** 3 / wall / 1e12, 3))
        for k in ("sbr_ms", "bc_ms", "solver_ms", "sbr_back_ms", "bc_back_ms", "final_ms"):
            v = getattr(st, k)
            rec[k] = [round(v[0], 2), round(v[1], 2), round(v[1] - v[0], 2)]
        out.append(rec)
        print(json.dumps(rec), flush=True)
    if check:
        del ws, a
        torch.cuda.empty_cache()
        # Q is column-major in a (n, n) row-major tensor -> q.t() is the matrix
        Q = q.t()
        R = a0 @ Q
        R -= Q * lam
        res = (torch.linalg.norm(R) / (n * torch.linalg.norm(a0))).item()
        del R
        torch.cuda.empty_cache()
        E = Q.t() @ Q
        E.diagonal().sub_(1.0)
        orth = (torch.linalg.norm(E) / n).item()
        print(json.dumps(dict(n=n, residual=res, ortho=orth)), flush=True)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("ns", type=int, nargs="+")
    ap.add_argument("--b", type=int, default=32)
    ap.add_argument("--order", default="pipelined")
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    for n in args.ns:
        run(n, args.b, args.order, args.check, args.reps)
        torch.cuda.empty_cache()
