"""One GEMM of a given shape through cuBLAS (torch) and through libpevd, for an ncu capture:
  ncu --metrics ... python tools/gemm_shape_ncu.py M N K beta"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_16174_b200 import _lib  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1:4])
beta = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0
A = torch.randn(m, k, dtype=torch.float64, device="cuda")
B = torch.randn(k, n, dtype=torch.float64, device="cuda")
C = torch.randn(m, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    C.addmm_(A, B, beta=beta, alpha=-1.0)
L = _lib.load()
P = ctypes.c_void_p
Af = torch.randn(m * k, dtype=torch.float64, device="cuda")
Bf = torch.randn(k * n, dtype=torch.float64, device="cuda")
Cf = torch.randn(m * n, dtype=torch.float64, device="cuda")
ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
for _ in range(2):
    _lib.check(L.pevd_dgemm(0, 0, m, n, k, -1.0, P(Af.data_ptr()), m, P(Bf.data_ptr()), k, beta,
                            P(Cf.data_ptr()), m, P(ws.data_ptr()), ws.numel(),
                            P(torch.cuda.current_stream().cuda_stream)), "gemm")
torch.cuda.synchronize()
