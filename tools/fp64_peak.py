"""FP64 roofline denominators on this B200: cuBLAS DGEMM (via torch) burst + sustained.

Reference measurement only (the product never calls cuBLAS); results -> profiles/fp64_peaks.json.
"""
import json, subprocess, sys, time
import torch

def dgemm(n, secs=None, reps=10):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 0.0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if secs is None:
        for _ in range(reps):
            e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
            best = max(best, 2 * n**3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
        return best
    t0 = time.time(); cnt = 0
    e0.record()
    while time.time() - t0 < secs:
        torch.matmul(a, b); cnt += 1
        if cnt % 4 == 0:
            torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    return 2 * n**3 * cnt / (e0.elapsed_time(e1) * 1e-3) / 1e12

if __name__ == "__main__":
    res = {"cublas_dgemm_8192_burst_tflops": dgemm(8192),
           "cublas_dgemm_8192_sustained_4s_tflops": dgemm(8192, secs=4.0)}
    out = subprocess.run(["./tools/fp64_peak"], capture_output=True, text=True).stdout
    res["micro"] = [json.loads(l) for l in out.splitlines() if l.strip()]
    res["gpu"] = torch.cuda.get_device_name(0)
    print(json.dumps(res, indent=1))
    with open("gpurun_out/fp64_peaks.json", "w") as f:
        json.dump(res, f, indent=1)
