"""Generate golden fixtures from the REAL reference package (`pipeevd`).

Run in the build container, where /root/reference exists:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Writes tests/golden/golden.npz.  The GPU box never runs this (the reference is
not there); tests only read the committed .npz.
"""
import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import pipeevd  # noqa: E402
from pipeevd import (BandMatrix, PipelineConfig, SbrConfig, SymmetricMatrix,  # noqa: E402
                     TridiagonalMatrix, back_plan_sizes, bc_back_apply, bc_reduce,
                     comm_broadcast_words, comm_triangular_words, crossover_bandwidth,
                     house_vector, make_back_plan, partition, run, sbr_reduce,
                     tridiag_eig)
from pipeevd.matgen import KINDS, SpectrumSpec, generate  # noqa: E402
from pipeevd.sbr import round_schedule  # noqa: E402

out = {}


def put(key, val):
    out[key] = np.asarray(val)


# ---- known-answer tests (reference tests cite these) ----
for idx, x in enumerate(([0.0, 3.0, 4.0], [3.5, 0.0, 0.0], [-2.0, 1.0, 2.0], [0.0, 0.0, 0.0],
                         [1e-300, 1e-300, 0.0], [5.0])):
    v, tau, alpha = house_vector(np.array(x))
    put(f"hv{idx}_x", x); put(f"hv{idx}_v", v); put(f"hv{idx}_tau", tau); put(f"hv{idx}_alpha", alpha)

put("rs_12_4", round_schedule(12, 4)); put("rs_11_4", round_schedule(11, 4))
put("rs_100_32", round_schedule(100, 32))
put("part_10_3", partition(10, 3)); put("part_49152_8", partition(49152, 8))
put("plan_8192_4", make_back_plan(8192, 4, 2048, 0.05).sizes)
put("bps_49152_8_05", back_plan_sizes(49152, 8, 0.05))
put("bps_10_3_05", back_plan_sizes(10, 3, 0.05))
put("cbw_8_2", comm_broadcast_words(8, 2)); put("ctw_8_2", comm_triangular_words(8, 2))
put("cbw_91_7", comm_broadcast_words(91, 7))
put("cross", crossover_bandwidth(1e13, 0.35e12))

# ---- SBR: dense -> band ----
sbr_cases = [(12, 4, 0), (11, 4, 1), (40, 4, 2), (64, 8, 3), (91, 7, 4), (128, 32, 5)]
for idx, (n, b, seed) in enumerate(sbr_cases):
    g = np.random.default_rng(seed).standard_normal((n, n))
    a = (g + g.T) / 2
    band, fac = sbr_reduce(SymmetricMatrix.from_dense(a), SbrConfig(b=b))
    put(f"sbr{idx}_nb", [n, b]); put(f"sbr{idx}_a", a); put(f"sbr{idx}_bands", band.bands)
    p0 = fac.panels[0]
    put(f"sbr{idx}_w0", p0.W); put(f"sbr{idx}_y0", p0.Y)
    pl = fac.panels[-1]
    put(f"sbr{idx}_wl", pl.W); put(f"sbr{idx}_yl", pl.Y)
    put(f"sbr{idx}_npanels", len(fac.panels))

# ---- BC: band -> tridiagonal ----
bc_cases = [(10, 2, 10), (24, 3, 11), (40, 4, 12), (64, 8, 13), (100, 16, 14), (130, 32, 15)]
for idx, (n, b, seed) in enumerate(bc_cases):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n)); a = (a + a.T) / 2
    band = BandMatrix.from_dense(np.tril(np.triu(a, -b), b), b)
    t, u = bc_reduce(band)
    put(f"bc{idx}_nb", [n, b]); put(f"bc{idx}_bands", band.bands)
    put(f"bc{idx}_d", t.d); put(f"bc{idx}_e", t.e)
    put(f"bc{idx}_i", u.i_idx); put(f"bc{idx}_j", u.j_idx); put(f"bc{idx}_row0", u.row0)
    put(f"bc{idx}_len", u.length); put(f"bc{idx}_tau", u.tau); put(f"bc{idx}_v", u.v)
    x = rng.standard_normal((n, 5))
    put(f"bc{idx}_x", x)
    put(f"bc{idx}_qbtx", bc_back_apply(u, x, direction="reordered"))
    put(f"bc{idx}_qbx", bc_back_apply(u, x, direction="conventional"))

# ---- tridiagonal solver ----
td_cases = [(1, 20), (2, 21), (7, 22), (33, 23), (80, 24)]
for idx, (n, seed) in enumerate(td_cases):
    rng = np.random.default_rng(seed)
    d = rng.standard_normal(n); e = rng.standard_normal(max(n - 1, 0))
    r = tridiag_eig(TridiagonalMatrix(d, e), want_vectors=True)
    put(f"td{idx}_d", d); put(f"td{idx}_e", e); put(f"td{idx}_lam", r.lam); put(f"td{idx}_q", r.Q)
# graded / clustered tridiagonals
d = np.array([1e6] + [1e-2] * 30); e = np.full(30, 1e-3)
r = tridiag_eig(TridiagonalMatrix(d, e), want_vectors=True)
put("tdc_d", d); put("tdc_e", e); put("tdc_lam", r.lam); put("tdc_q", r.Q)

# ---- whole pipeline ----
run_cases = [(48, 8, 1, "pipelined", 31), (64, 8, 2, "pipelined", 32), (64, 8, 4, "conventional", 33),
             (96, 32, 1, "pipelined", 34), (40, 4, 3, "sequential", 35)]
for idx, (n, b, w, order, seed) in enumerate(run_cases):
    g = np.random.default_rng(seed).standard_normal((n, n))
    a = (g + g.T) / 2
    res, events, ledger, counter = run(a, PipelineConfig(workers=w, b=b, order=order))
    put(f"run{idx}_cfg", [n, b, w, seed]); put(f"run{idx}_order", order)
    put(f"run{idx}_a", a); put(f"run{idx}_lam", res.lam); put(f"run{idx}_q", res.Q)
    put(f"run{idx}_sbr_words", ledger.words(stage="SBR"))
    put(f"run{idx}_bc_words", ledger.words(stage="BC"))
    put(f"run{idx}_macs", [counter.by_stage.get(s, 0) for s in
                           ("SBR", "BC", "Solver", "SBR-Back", "BC-Back", "FinalMultiply")])

# six planted spectra (matgen.py) at n=64, seed 1 -- A itself is stored
for idx, kind in enumerate(KINDS):
    a, lam = generate(SpectrumSpec(kind, 64, seed=1))
    put(f"spec{idx}_kind", kind); put(f"spec{idx}_a", a.data); put(f"spec{idx}_lam", lam)
    res, _, _, _ = run(a, PipelineConfig(workers=2, b=8))
    put(f"spec{idx}_runlam", res.lam)

path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
np.savez_compressed(path, **out)
print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")
