import sys, ctypes, torch
sys.path.insert(0, ".")
from paper_2511_16174_b200 import _lib
L = _lib.load(); P = ctypes.c_void_p
n, b = int(sys.argv[1]), 32
g = torch.Generator(device="cuda"); g.manual_seed(0)
bands = torch.randn((b + 1) * n, dtype=torch.float64, device="cuda", generator=g)
nref = L.pevd_bc_num_reflectors(n, b)
tau = torch.empty(nref, dtype=torch.float64, device="cuda"); V = torch.empty(nref * 32, dtype=torch.float64, device="cuda")
d = torch.empty(n, dtype=torch.float64, device="cuda"); e = torch.empty(n, dtype=torch.float64, device="cuda")
ws = torch.empty(L.pevd_bc_workspace_bytes(n, b), dtype=torch.uint8, device="cuda")
s = P(torch.cuda.current_stream().cuda_stream)
_lib.check(L.pevd_bc(n, b, P(bands.data_ptr()), P(d.data_ptr()), P(e.data_ptr()), P(tau.data_ptr()), P(V.data_ptr()), 32, P(ws.data_ptr()), s), "bc")
X = torch.randn((n, n), dtype=torch.float64, device="cuda")
ws = torch.empty(L.pevd_bc_back_workspace_bytes(n, n, 32), dtype=torch.uint8, device="cuda")
_lib.check(L.pevd_bc_back_left(n, b, P(tau.data_ptr()), P(V.data_ptr()), 32, P(X.data_ptr()), n, n, P(ws.data_ptr()), s), "bcbl")
torch.cuda.synchronize()
