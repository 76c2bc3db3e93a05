"""Time the UNMODIFIED reference package (`pipeevd`, installed into baseline/_ref by
`pip install --target baseline/_ref`) on this host's cores: pipeevd.run(A, PipelineConfig(...))
through its own public API (reference pipeline.py:511-548), with the harness patch SURVEY.md §8(c)
names (`_recv` timeout raised so big n does not abort).  Used by bench.py --impl reference and by
the per-stage n^3 extrapolation to n = 49152:

    python tools/ref_cpu.py --ns 1024 2048 4096 --workers 1 8 > profiles/r02_reference_cpu.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def load_reference():
    """Import pipeevd from baseline/_ref (never from /root/reference: it does not exist on the
    GPU box).  Raises ImportError when the install is missing."""
    if not os.path.isdir(os.path.join(REF, "pipeevd")):
        raise ImportError(f"reference not installed in {REF}")
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "pevd_numba_cache"))
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import pipeevd
    from pipeevd import pipeline
    pipeline._recv.__defaults__ = (1e7,)  # the 120 s hand-off timeout aborts big n
    return pipeevd


def goe(n: int, seed: int):
    import numpy as np
    g = np.random.default_rng(seed).standard_normal((n, n))
    return (g + g.T) / 2


def time_run(pipeevd, a, workers: int, b: int = 32, want_vectors: bool = True):
    """One reference EVD; returns (wall seconds, per-stage busy seconds summed over lanes)."""
    t0 = time.perf_counter()
    res, events, _, _ = pipeevd.run(a, pipeevd.PipelineConfig(workers=workers, b=b,
                                                              want_vectors=want_vectors))
    wall = time.perf_counter() - t0
    stages = {}
    for e in events:
        stages[e.stage] = stages.get(e.stage, 0.0) + e.duration / 1e9
    return wall, stages, res


def host_info():
    info = {"cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["model"] = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        from threadpoolctl import threadpool_info
        info["blas_threads"] = [p.get("num_threads") for p in threadpool_info()
                                if p.get("user_api") == "blas"]
    except Exception:
        pass
    return info


def warm(pipeevd, workers=(1,)):
    a = goe(256, 256)
    for w in workers:
        time_run(pipeevd, a, w)


def extrapolate(rows, n_target: int):
    """Per-stage n^3 fit through the largest measured n (the stages are O(n^3) or, for the
    chase, O(n^2 b) -- scaling it by n^3 over-estimates it, which favours the reference)."""
    best = max(rows, key=lambda r: r["n"])
    s = (n_target / best["n"]) ** 3
    return {"from_n": best["n"], "workers": best["workers"], "scale": s,
            "wall_s": best["wall_s"] * s,
            "stages_s": {k: v * s for k, v in best["stages_s"].items()}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", type=int, nargs="+", default=[1024, 2048, 4096])
    ap.add_argument("--workers", type=int, nargs="+", default=[1, os.cpu_count() or 1])
    ap.add_argument("--target", type=int, default=49152)
    args = ap.parse_args()
    pipeevd = load_reference()
    warm(pipeevd, args.workers)
    rows = []
    for n in args.ns:
        a = goe(n, n)
        for w in args.workers:
            if w > n:
                continue
            wall, stages, _ = time_run(pipeevd, a, w)
            rows.append({"n": n, "workers": w, "wall_s": round(wall, 3),
                         "tflops": 4 * n ** 3 / wall / 1e12,
                         "stages_s": {k: round(v, 3) for k, v in stages.items()}})
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    out = {"host": host_info(), "rows": rows,
           "extrapolated": {str(w): extrapolate([r for r in rows if r["workers"] == w], args.target)
                            for w in args.workers if any(r["workers"] == w for r in rows)}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
