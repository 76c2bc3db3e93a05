"""Host<->device copy paths for run()'s numpy buffers at n = 49152 (19.3 GB): pageable
torch copy, cudaHostRegister in place, and multi-threaded staging through pinned chunks."""
import ctypes
import json
import sys
import threading
import time

import numpy as np
import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 49152
a = np.empty((n, n))
a[:] = 1.0
out = {}
t = time.perf_counter(); d = torch.from_numpy(a).cuda(); torch.cuda.synchronize(); out["pageable_h2d_s"] = time.perf_counter() - t
t = time.perf_counter(); d.cpu(); out["pageable_d2h_s"] = time.perf_counter() - t
cr = torch.cuda.cudart()
t = time.perf_counter(); rc = cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0); out["register_s"] = time.perf_counter() - t
out["register_rc"] = int(rc)
ta = torch.from_numpy(a)
t = time.perf_counter(); d.copy_(ta, non_blocking=True); torch.cuda.synchronize(); out["registered_h2d_s"] = time.perf_counter() - t
t = time.perf_counter(); ta.copy_(d, non_blocking=True); torch.cuda.synchronize(); out["registered_d2h_s"] = time.perf_counter() - t
t = time.perf_counter(); cr.cudaHostUnregister(a.ctypes.data); out["unregister_s"] = time.perf_counter() - t
# staged, 4 threads x 2 pinned chunks of 256 MB
def staged(src, dst, nthreads=4, chunk=1 << 25):
    flat_s = torch.from_numpy(src).view(-1)
    flat_d = dst.view(-1)
    N = flat_s.numel()
    def work(tid):
        st = torch.cuda.Stream()
        bufs = [torch.empty(chunk, dtype=torch.float64, pin_memory=True) for _ in range(2)]
        evs = [None, None]
        k = 0
        for c0 in range(tid * chunk, N, nthreads * chunk):
            c1 = min(N, c0 + chunk)
            b = bufs[k & 1]
            if evs[k & 1] is not None:
                evs[k & 1].synchronize()
            b[: c1 - c0].copy_(flat_s[c0:c1])
            with torch.cuda.stream(st):
                flat_d[c0:c1].copy_(b[: c1 - c0], non_blocking=True)
                e = torch.cuda.Event(); e.record(st); evs[k & 1] = e
            k += 1
        st.synchronize()
    th = [threading.Thread(target=work, args=(i,)) for i in range(nthreads)]
    [x.start() for x in th]; [x.join() for x in th]
for nt in (4, 8):
    t = time.perf_counter(); staged(a, d, nt); torch.cuda.synchronize(); out[f"staged{nt}_h2d_s"] = time.perf_counter() - t
print(json.dumps({k: round(v, 3) if isinstance(v, float) else v for k, v in out.items()}))
