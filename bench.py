"""Benchmark: FP64 EVD TFLOP/s (4 n^3 / wall, eigenvectors) at n = 49152 on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--n 49152]

One step = one full two-stage EVD with eigenvectors of a synthetic random symmetric matrix
(A = (G + G^T)/2, G ~ N(0,1) from a seeded torch generator on the device).  `value` times the
device-resident path (pevd_syevd_device, input already in HBM; A is 19.3 GB, far larger than the
126 MB L2, so no L2 flush is needed); `e2e` times the C-ABI call with HOST buffers
(pevd_syevd: pinned host A in, lambda and Q out, device allocation included).  Under torchrun
(N > 1) the N ranks solve ONE EVD together (blockwise columns, csrc/dist.cu over NCCL) and
value = 4 n^3 / max-over-ranks time; a failure there exits non-zero (no replica fallback).

--impl reference times the reference package itself (pipeevd.run, installed unmodified into
baseline/_ref, tools/ref_cpu.py) on a bounded sample (n=1024 per step) on the host's cores.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 EVD TFLOPS + wall time (n=49152, with eigvecs) at 1/2/4/8 B200"


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev, self.rows, self._stop = dev, [], threading.Event()
        self._th = threading.Thread(target=self._loop, daemon=True)

    def _loop(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.25)

    def __enter__(self):
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def stage_flops(n: int, order: str = "conventional"):
    """Algorithmic FP64 flops per stage; BC-Back as its BLAS2 count.
    SBR-Back forms Q_s ((4/3) n^3, pipelined/sequential) or applies it to Q_d from the left
    (2 n^3, conventional, which has no final GEMM)."""
    conv = order == "conventional"
    return {"sbr": 4 * n ** 3 / 3, "sbr_back": (2 if conv else 4 / 3) * n ** 3,
            "bc_back": 2 * n ** 3, "final": 0 if conv else 2 * n ** 3, "solver": 4 * n ** 3 / 3}


def run_b200(args):
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1 or args.blockwise:
        # one EVD over all ranks (csrc/dist.cu over NCCL); a failure is a failure, no fallback
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29513")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local), rank=rank,
                                    world_size=world)
        return run_b200_distributed(args)
    return run_b200_single(args)


def stage_roofline(n, b, stage_ms, flops_exec, order, peaks, G=1):
    """Per-stage roofline: achieved rate / (G x peak) for each of the five stages.
    GEMM-like stages: algorithmic flops on the FP64 DMMA peak; the divide and
    conquer: the merge-GEMM flops it EXECUTED (deflation-dependent, summed on the device); the
    bulge chase: its compulsory HBM bytes on the measured HBM bandwidth."""
    fl = stage_flops(n, order)
    nref = sum(n - 2 - j * b for j in range((n - 3) // b + 1)) if n >= 3 else 0
    bc_bytes = 8 * ((b + 1) * n + nref * (((b + 7) // 8) * 8 + 1) + 2 * n)
    out = {}
    for k, alg in (("sbr", fl["sbr"]), ("sbr_back", fl["sbr_back"]), ("bc_back", fl["bc_back"]),
                   ("final", fl["final"]), ("solver", flops_exec.get("solver", 0.0))):
        t = stage_ms.get(k, 0.0)
        if t <= 0 or alg <= 0:
            continue
        ach = alg / (t * 1e-3) / 1e12
        out[k] = {"bound": "tensor", "achieved": round(ach, 3), "peak": round(G * peaks["dmma"], 2),
                  "unit": "TFLOP/s", "frac": round(ach / (G * peaks["dmma"]), 4),
                  "ms": round(t, 1), "flops": alg,
                  "flops_executed": flops_exec.get(k)}
    t = stage_ms.get("bc", 0.0)
    if t > 0:
        hbm = peaks["hbm_gbs"]
        ach = bc_bytes / (t * 1e-3) / 1e9
        out["bc"] = {"bound": "hbm (latency-bound chase)", "achieved": round(ach, 2),
                     "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 5), "ms": round(t, 1),
                     "bytes": bc_bytes,
                     "note": "compulsory bytes 8[(b+1)n + N_refl(pad8(b)+1) + 2n]; the chase is "
                             "one GPU's wavefront (replicated partitions relay across GPUs)"}
    return out


def run_b200_distributed(args):
    """N ranks cooperate on ONE n x n EVD: blockwise columns (csrc/dist.cu over NCCL)."""
    import ctypes
    import torch
    import torch.distributed as dist
    from paper_2511_16174_b200 import PipelineConfig, _lib
    from paper_2511_16174_b200.distributed import run_distributed
    from paper_2511_16174_b200.schedule import partition
    from paper_2511_16174_b200.pipeline import back_ranges
    rank, world, local = dist_env()
    L = _lib.load()
    n, b = args.n, args.b
    c0w, c1w = partition(n, world)[rank]
    r0, r1 = back_ranges(n, world, 0.0)[rank]
    g = torch.Generator(device="cuda")
    g.manual_seed(args.seed)          # every rank generates the same A, keeps its columns
    a0 = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    a0.add_(a0.t().clone())
    a0.mul_(0.5)
    blk0 = a0[c0w:c1w].clone()        # (w, n): column-major n x w, this rank's columns
    del a0
    torch.cuda.empty_cache()
    cfg = PipelineConfig(workers=world, b=b, order=args.order)
    blk = torch.empty_like(blk0)

    def block(c0, c1):
        return blk

    def barrier():
        dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        blk.copy_(blk0)
        run_distributed(block, cfg, n=n, gather_q=False)
    launches0 = L.pevd_kernel_launches()
    times, infos = [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            blk.copy_(blk0)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _, _, ledger, info = run_distributed(block, cfg, n=n, gather_q=False)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            infos.append(info)
            barrier()
    launches = (L.pevd_kernel_launches() - launches0) // max(1, args.steps)
    ms = sum(times) / len(times)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = 4 * n ** 3 / (ms * 1e-3) / 1e12
    # per-stage times: the max over ranks of each stage's span; executed flops summed
    st = infos[-1]["stats"].stages
    mine = [getattr(st, k + "_ms")[1] - getattr(st, k + "_ms")[0]
            for k in ("sbr", "bc", "solver", "sbr_back", "bc_back", "final")] + list(st.flops)
    tt = torch.tensor(mine, dtype=torch.float64, device="cuda")
    mx = tt[:6].clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = tt[6:].clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    names = ("sbr", "bc", "solver", "sbr_back", "bc_back", "final")
    stage_ms = dict(zip(names, mx.tolist()))
    fx = dict(zip(("sbr", "bc", "sbr_back", "bc_back", "solver", "final"), sm.tolist()))
    # the divide and conquer is replicated (every rank solves): one rank's executed flops
    fx["solver"] = fx["solver"] / world
    peaks = load_fp64_peaks()
    stages = stage_roofline(n, b, stage_ms, fx, args.order, peaks, world)
    dom = max((k for k in stages if k != "bc"), key=lambda k: stages[k]["ms"])
    roofline = dict(stages[dom])
    roofline.update({"kernel": dom, "traffic": None,
                     "peak_source": f"{world} x FP64 DMMA microbenchmark "
                                    f"(profiles/r01_fp64_peaks.json)",
                     "stages": stages,
                     "comm_words": ledger.total_words,
                     "comm_words_by_stage": {k: ledger.words(stage=k) for k in ledger.stages()}})
    clocks = clk.summary()
    # ---- e2e: this rank's column block from pinned host memory, its Q slab back to the host
    e2e = None
    if not args.no_e2e:
        hblk = torch.empty(blk0.shape, dtype=torch.float64, pin_memory=True)
        hblk.copy_(blk0)
        hq = torch.empty((max(r1 - r0, 1), n), dtype=torch.float64, pin_memory=True)
        del blk0
        torch.cuda.empty_cache()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        blk.copy_(hblk, non_blocking=True)
        res, _, _, info = run_distributed(block, cfg, n=n, gather_q=False)
        hq.copy_(info["q_part"], non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        ems = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        ems = float(ems.item())
        e2e = {"value": round(4 * n ** 3 / (ems * 1e-3) / 1e12, 4), "unit": "TFLOP/s",
               "ms_per_step": round(ems, 1), "h2d_bytes_per_step": 8 * n * n,
               "d2h_bytes_per_step": 8 * n * n,
               "note": "each rank: its column block pinned host -> device, its Q slab back"}
    cpu = cpu_baseline(args.cpu_n) if (rank == 0 and not args.no_cpu) else None
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 4), "unit": "TFLOP/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 1),
                "wall_s_per_evd": round(ms / 1e3, 3), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"ONE dense symmetric FP64 EVD with eigenvectors, n={n}, "
                                       f"b={b}, order={args.order}, blockwise columns over "
                                       f"{world} GPUs (csrc/dist.cu, NCCL)",
                           "n": n, "b": b, "order": args.order, "parallelism": f"blockwise{world}",
                           "l2": "input >> 126 MB L2 (no flush needed)",
                           "flop_convention": "4 n^3 / wall (PAPER.md:92)"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "clocks": clocks, "gpu_launches": int(launches), "impl": "b200"}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def run_b200_single(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2511_16174_b200 import _lib

    rank, world, local = dist_env()
    L = _lib.load()
    n, b = args.n, args.b
    oc = _lib.ORDER_CODES[args.order]
    g = torch.Generator(device="cuda")
    g.manual_seed(args.seed + rank)
    a0 = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    a0.add_(a0.t().clone())
    a0.mul_(0.5)
    a = torch.empty_like(a0)
    q = torch.empty_like(a0)
    lam = torch.empty(n, dtype=torch.float64, device="cuda")
    ws_bytes = L.pevd_syevd_workspace_bytes(n, b, 1, oc)
    a0_host = None
    if ws_bytes + (2 << 30) > torch.cuda.mem_get_info()[0]:
        # pipelined / sequential order at n = 49152 need a 125 GB workspace: the pristine copy of
        # A used to reset the (destroyed) input between steps then lives in pinned host memory
        # (the reset is outside the timed region)
        a0_host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        a0_host.copy_(a0)
        del a0
        torch.cuda.empty_cache()
        a0 = None
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    a_src = a0 if a0_host is None else a0_host
    stream = torch.cuda.current_stream()
    P = ctypes.c_void_p

    def step(st):
        rc = L.pevd_syevd_device(n, b, P(a.data_ptr()), n, P(lam.data_ptr()), P(q.data_ptr()), n,
                                 1, oc, P(ws.data_ptr()), ws.numel(), P(stream.cuda_stream),
                                 ctypes.byref(st))
        _lib.check(rc, "pevd_syevd_device")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        a.copy_(a_src)
        step(_lib.PevdStats())
    times, stats = [], []
    launches0 = L.pevd_kernel_launches()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            a.copy_(a_src)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            st = _lib.PevdStats()
            e0.record(stream)
            step(st)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            stats.append(st)
            barrier()
    launches = (L.pevd_kernel_launches() - launches0) // max(1, args.steps)
    ms = sum(times) / len(times)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * 4 * n ** 3 / (ms * 1e-3) / 1e12

    # accuracy of the last step's result on the device (outside the timed region; verification):
    # north-star residual ||A Q - Q Lam||_F / (n ||A||_F) and orthogonality ||Q^T Q - I||_F / n
    accuracy = None
    if not args.no_check:
        from paper_2511_16174_b200 import matgen
        if a0 is None:  # A back on the device for the check (the workspace is no longer needed)
            del ws
            ws = None
            torch.cuda.empty_cache()
            a0 = a0_host.to("cuda")
        res, orth = matgen.accuracy(a0, lam, q)
        accuracy = {"residual": res, "orthogonality": orth, "bound": 1e-12,
                    "pass": bool(res <= 1e-12 and orth <= 1e-12)}
    # stage breakdown of the last step (CUDA events on the launching streams, inside the lib)
    st = stats[-1]
    stage_ms = {k: getattr(st, k + "_ms")[1] - getattr(st, k + "_ms")[0]
                for k in ("sbr", "bc", "solver", "sbr_back", "bc_back", "final")}
    fx = dict(zip(("sbr", "bc", "sbr_back", "bc_back", "solver", "final"), list(st.flops)))
    fl = stage_flops(n, args.order)
    dom = max(("sbr", "sbr_back", "bc_back", "final", "solver"), key=lambda k: stage_ms[k])
    peaks = load_fp64_peaks()
    peak = peaks["dmma"]  # every GEMM-like stage (BC-Back included) runs on DMMA
    achieved = fl[dom] / (stage_ms[dom] * 1e-3) / 1e12
    traffic, traffic_src = None, None
    try:  # dram bytes of that kernel's launch from the committed ncu capture (same n only)
        tr = json.load(open(os.path.join(ROOT, "profiles", "r02_traffic.json"))).get(dom)
        if tr and tr.get("n") == n:
            traffic = tr["dram_read_bytes"] + tr["dram_write_bytes"]
            traffic_src = "profiles/r02_traffic.json (ncu dram__bytes_read+write, one launch)"
    except Exception:
        pass
    roofline = {"bound": "tensor", "kernel": dom, "achieved": round(achieved, 3),
                "peak": peak, "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
                "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": "FP64 DMMA (mma.sync m8n8k4) microbenchmark"
                               " on this pool's B200 (profiles/r01_fp64_peaks.json); "
                               "MEASURED_PEAKS.json has no FP64 entry",
                "stage_ms": {k: round(v, 1) for k, v in stage_ms.items()},
                "stages": stage_roofline(n, b, stage_ms, fx, args.order, peaks),
                "executed_flops": {k: v for k, v in fx.items() if v > 0}}
    clocks = clk.summary()

    # ---- e2e through the C ABI with host buffers (pevd_syevd)
    e2e = None
    if not args.no_e2e:
        a_host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        a_host.copy_(a0 if a0 is not None else a0_host)
        del a, q, ws
        a0 = a0_host = a_src = None  # the library allocates its own A, Q and workspace
        torch.cuda.empty_cache()
        q_host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        lam_host = torch.empty(n, dtype=torch.float64, pin_memory=True)
        barrier()
        t0 = time.perf_counter()
        rc = L.pevd_syevd(n, b, P(a_host.data_ptr()), n, P(lam_host.data_ptr()),
                          P(q_host.data_ptr()), n, 1, oc, ctypes.byref(_lib.PevdStats()))
        t1 = time.perf_counter()
        _lib.check(rc, "pevd_syevd")
        ems = (t1 - t0) * 1e3
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        # pevd_syevd uploads the lower trapezoid of each 512-column block (include/pevd.h:
        # only the lower triangle of A is read) and downloads Q slab by slab, overlapped with
        # the last SBR-Back blocks (csrc/hostio.h)
        h2d = sum(8 * (n - j0) * min(512, n - j0) for j0 in range(0, n, 512))
        e2e = {"value": round(world * 4 * n ** 3 / (ems * 1e-3) / 1e12, 4), "unit": "TFLOP/s",
               "ms_per_step": round(ems, 1), "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 8 * n * n + 8 * n}
    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_baseline(args.cpu_n)
    same_n = None
    if rank == 0 and not args.no_same_n:
        same_n = same_n_runs(L, b, args.order, (1024, 4096))
        if cpu and cpu.get("kind") == "reference" and "1024" in same_n:
            same_n["ratio_vs_reference_n1024"] = round(same_n["1024"]["tflops"] / cpu["value"], 1)
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 4), "unit": "TFLOP/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 1),
                "wall_s_per_evd": round(ms / 1e3, 3), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"dense symmetric FP64 EVD with eigenvectors, n={n}, b={b}, "
                                       f"order={args.order}, A=(G+G^T)/2 G~N(0,1)",
                           "n": n, "b": b, "order": args.order,
                           "parallelism": "1 GPU",
                           "l2": "input 8n^2 = %.1f GB >> 126 MB L2 (no flush needed)" % (8 * n * n / 1e9),
                           "flop_convention": "4 n^3 / wall (PAPER.md:92)"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
                "accuracy": accuracy, "same_n": same_n,
                "gpu_launches": int(launches), "impl": "b200"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def same_n_runs(L, b, order, ns):
    """The same device path at the reference arm's sizes (a like-for-like ratio beside the
    headline): best of 3 CUDA-event-timed EVDs per n, inputs resident."""
    import ctypes
    import torch
    from paper_2511_16174_b200 import _lib
    out = {}
    oc = _lib.ORDER_CODES[order]
    P = ctypes.c_void_p
    for n in ns:
        g = torch.Generator(device="cuda")
        g.manual_seed(n)
        a0 = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
        a0 = (a0 + a0.t()) * 0.5
        a = torch.empty_like(a0)
        q = torch.empty_like(a0)
        lam = torch.empty(n, dtype=torch.float64, device="cuda")
        ws = torch.empty(L.pevd_syevd_workspace_bytes(n, b, 1, oc), dtype=torch.uint8, device="cuda")
        s = torch.cuda.current_stream()
        best = None
        for _ in range(4):
            a.copy_(a0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            _lib.check(L.pevd_syevd_device(n, b, P(a.data_ptr()), n, P(lam.data_ptr()),
                                           P(q.data_ptr()), n, 1, oc, P(ws.data_ptr()),
                                           ws.numel(), P(s.cuda_stream),
                                           ctypes.byref(_lib.PevdStats())), "same_n")
            e1.record(s)
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1)
            best = t if best is None else min(best, t)
        out[str(n)] = {"ms": round(best, 2), "tflops": round(4 * n ** 3 / (best * 1e-3) / 1e12, 4)}
    return out


def load_fp64_peaks():
    path = os.path.join(ROOT, "profiles", "r01_fp64_peaks.json")
    try:
        d = json.load(open(path))
        dmma = max(x["tflops"] for x in d["micro"] if x["kind"].startswith("dmma"))
        dfma = max(x["tflops"] for x in d["micro"] if x["kind"] == "dfma")
        out = {"dmma": round(dmma, 2), "dfma": round(dfma, 2),
               "cublas_dgemm": round(d.get("cublas_dgemm_8192_sustained_4s_tflops", 0), 2)}
    except Exception:
        out = {"dmma": 37.17, "dfma": 34.19, "cublas_dgemm": 35.41}
    try:  # HBM: the driver-measured copy bandwidth of this pool's B200
        out["hbm_gbs"] = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        out["hbm_gbs"] = 6440.1
    return out


def cpu_baseline(n_cpu: int):
    """The reference package itself (pipeevd.run from baseline/_ref, its own public API, 1 worker
    thread -- the fastest setting at this size -- plus OpenBLAS on all host threads) on this host:
    one EVD with vectors at n_cpu.  Falls back to the oracle port only when the install is
    missing, and says so in `kind`."""
    import numpy as np
    try:
        from tools.ref_cpu import goe, load_reference, time_run, warm
        pipeevd = load_reference()
        warm(pipeevd)
        a = goe(n_cpu, n_cpu)
        dt, stages, _ = time_run(pipeevd, a, 1)
        return {"value": round(4 * n_cpu ** 3 / dt / 1e12, 6), "unit": "TFLOP/s",
                "cores": os.cpu_count(), "kind": "reference",
                "sample": f"pipeevd.run (baseline/_ref, unmodified) n={n_cpu} with vectors, "
                          f"workers=1 (+ OpenBLAS threads), {dt:.2f} s"}
    except ImportError:
        from oracle import oracle as orc
        g = np.random.default_rng(n_cpu).standard_normal((n_cpu, n_cpu))
        a = (g + g.T) / 2
        orc.evd(a[:64, :64], 32, True)  # warm the library
        t0 = time.perf_counter()
        orc.evd(a, 32, True)
        dt = time.perf_counter() - t0
        return {"value": round(4 * n_cpu ** 3 / dt / 1e12, 6), "unit": "TFLOP/s",
                "cores": os.cpu_count(), "kind": "port",
                "sample": f"one n={n_cpu} EVD with vectors (oracle/ port: the reference install is "
                          f"missing), {dt:.2f} s"}


def reference_extrapolation():
    """Committed per-stage n^3 extrapolation of the reference to n = 49152 (tools/ref_cpu.py on
    a GPU box host), labelled as such; None when absent."""
    path = os.path.join(ROOT, "profiles", "r02_reference_cpu.json")
    try:
        d = json.load(open(path))
        ex = {w: {"wall_s": round(v["wall_s"], 1), "from_n": v["from_n"],
                  "tflops": round(4 * 49152 ** 3 / v["wall_s"] / 1e12, 6)}
              for w, v in d["extrapolated"].items()}
        return {"source": "profiles/r02_reference_cpu.json (per-stage n^3 fit, extrapolated)",
                "host": d.get("host"), "by_workers": ex}
    except Exception:
        return None


def run_reference(args):
    """--impl reference: the unmodified reference package (pipeevd.run, baseline/_ref) on this
    host's cores, each step a bounded sample (n = --ref-n) of the workload."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from tools.ref_cpu import goe, host_info, load_reference, time_run, warm
    try:
        pipeevd = load_reference()
    except ImportError as exc:
        print(json.dumps({"impl": "reference", "unavailable": str(exc)}), flush=True)
        return
    n = args.ref_n
    workers = args.ref_workers
    warm(pipeevd, (workers,))
    a = goe(n, n)
    for _ in range(args.warmup):
        time_run(pipeevd, a, workers)
    ts, stages = [], None
    for _ in range(args.steps):
        dt, stages, _ = time_run(pipeevd, a, workers)
        ts.append(dt)
    dt = sum(ts) / len(ts)
    v = 4 * n ** 3 / dt / 1e12
    print(json.dumps({
        "metric": METRIC, "value": round(v, 6), "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": f"reference pipeevd.run with eigenvectors, bounded sample n={n} "
                               f"(b={args.b}, workers={workers}, order=pipelined: the reference "
                               f"default); n=49152 would take days on the host", "n": n,
                   "b": args.b, "workers": workers},
        "stage_busy_s": {k: round(x, 3) for k, x in (stages or {}).items()},
        "host": host_info(),
        "extrapolated_n49152": reference_extrapolation(),
        "cpu_baseline": {"value": round(v, 6), "unit": "TFLOP/s", "cores": os.cpu_count(),
                         "kind": "reference",
                         "sample": f"pipeevd.run n={n} with vectors per step, workers={workers} "
                                   f"(+ OpenBLAS on all host threads)"},
        "e2e": {"value": round(v, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=49152)
    ap.add_argument("--b", type=int, default=32)
    ap.add_argument("--order", default="conventional", choices=["pipelined", "sequential", "conventional"])
    ap.add_argument("--seed", type=int, default=49152)
    ap.add_argument("--cpu-n", type=int, default=1024)
    ap.add_argument("--ref-workers", type=int, default=1)
    ap.add_argument("--ref-n", type=int, default=1024)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true", help="skip the residual/orthogonality check")
    ap.add_argument("--no-same-n", action="store_true", help="skip the n=1024/4096 device runs")
    ap.add_argument("--blockwise", action="store_true",
                    help="run the distributed (csrc/dist.cu, NCCL) path even on one rank")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
