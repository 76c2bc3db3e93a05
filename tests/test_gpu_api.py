"""The reference's own end-to-end checks (pkg/tests/test_pipeline.py, test_acceptance.py),
run against the drop-in `run()` on the GPU, with the CPU oracle as the checker."""
import numpy as np
import pytest

import paper_2511_16174_b200 as pkg
from oracle import oracle as orc

pytestmark = pytest.mark.gpu
EPS = np.finfo(np.float64).eps


@pytest.fixture(scope="module")
def G():
    return np.load("tests/golden/golden.npz")


def _sym(n, seed):
    g = np.random.default_rng(seed).standard_normal((n, n))
    return (g + g.T) / 2


def test_small_problems_match_oracle():
    # test_pipeline.py:32-46 (Jacobi oracle -> the pinned oracle's eigenvalues)
    for seed in range(10):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(4, 40))
        workers = int(rng.integers(1, min(4, n) + 1))
        a = _sym(n, 100 + seed)
        res, events, ledger, counter = pkg.run(a, pkg.PipelineConfig(workers=workers, b=4))
        lam_ref = np.linalg.eigvalsh(a)
        np.testing.assert_allclose(res.lam, lam_ref, atol=1e-12 * np.abs(lam_ref).max())
        assert orc.backward_error(a, res.Q, res.lam) <= 1e-15
        assert orc.orthogonality(res.Q) <= 2 * EPS * 16


def test_golden_reference_runs(G):
    for idx in range(5):
        n, b, w, seed = (int(x) for x in G[f"run{idx}_cfg"])
        order = str(G[f"run{idx}_order"])
        a = G[f"run{idx}_a"]
        res, _, ledger, _ = pkg.run(a, pkg.PipelineConfig(workers=w, b=b, order=order))
        lam_ref = G[f"run{idx}_lam"]
        np.testing.assert_allclose(res.lam, lam_ref, atol=10 * n * EPS * np.abs(lam_ref).max())
        assert orc.backward_error(a, res.Q, res.lam) <= 1e-15
        assert orc.orthogonality(res.Q) <= 1e-15
        if w > 1:  # measured: one GPU moves nothing, G workers move the reference's SBR words
            assert ledger.words(stage="SBR") == int(G[f"run{idx}_sbr_words"])
            assert ledger.words(stage="BC") == int(G[f"run{idx}_bc_words"])
        else:
            assert ledger.total_words == 0
        # eigenvectors agree with the reference's up to sign for well separated eigenvalues
        q_ref = G[f"run{idx}_q"]
        gaps = np.minimum(np.r_[np.inf, np.diff(lam_ref)], np.r_[np.diff(lam_ref), np.inf])
        ok = gaps > 1e-6 * np.abs(lam_ref).max()
        dots = np.abs(np.sum(res.Q[:, ok] * q_ref[:, ok], axis=0))
        np.testing.assert_allclose(dots, 1.0, atol=1e-9)


def test_orders_agree():
    a = _sym(64, 5)
    results = {}
    for order in pkg.ORDERS:
        res, _, _, _ = pkg.run(a, pkg.PipelineConfig(workers=4, b=8, order=order))
        results[order] = res
        assert orc.backward_error(a, res.Q, res.lam) <= 1e-15
    for order in ("sequential", "conventional"):
        np.testing.assert_allclose(results[order].lam, results["pipelined"].lam,
                                   atol=1e-12 * np.abs(results["pipelined"].lam).max())


def test_reruns_bitwise_identical():
    a = _sym(200, 8)
    r1, _, _, _ = pkg.run(a, pkg.PipelineConfig(workers=3, b=8))
    r2, _, _, _ = pkg.run(a, pkg.PipelineConfig(workers=3, b=8))
    np.testing.assert_array_equal(r1.lam, r2.lam)
    np.testing.assert_array_equal(r1.Q, r2.Q)


def test_eigenvalues_only_mode():
    a = _sym(40, 11)
    r, _, _, _ = pkg.run(a, pkg.PipelineConfig(workers=2, b=4, want_vectors=False))
    assert r.Q is None and not r.vectors_computed
    full, _, _, _ = pkg.run(a, pkg.PipelineConfig(workers=2, b=4))
    np.testing.assert_allclose(r.lam, full.lam, atol=1e-14 * np.abs(full.lam).max())


def test_trace_file_and_counter(tmp_path):
    path = tmp_path / "trace.ndjson"
    a = _sym(48, 12)
    _, events, _, counter = pkg.run(a, pkg.PipelineConfig(workers=2, b=8, trace_path=str(path)))
    loaded = pkg.TraceLog.from_ndjson(path)
    assert loaded == events
    stages = {e.stage for e in loaded}
    assert {"SBR", "BC", "Solver", "BC-Back", "FinalMultiply"} <= stages
    # dependency contract of schedule.validate_trace: BC-Back after BC, Final after the solver
    end = {s: max(e.t_end for e in loaded if e.stage == s) for s in stages}
    start = {s: min(e.t_start for e in loaded if e.stage == s) for s in stages}
    assert start["BC-Back"] >= end["BC"] and start["FinalMultiply"] >= end["Solver"]
    for stage in ("SBR", "BC", "Solver", "SBR-Back", "BC-Back", "FinalMultiply"):
        assert counter.by_stage.get(stage, 0) > 0


def test_tiny_matrices():
    res, _, _, _ = pkg.run(np.array([[2.5]]), pkg.PipelineConfig(workers=1, b=4))
    np.testing.assert_array_equal(res.lam, [2.5])
    np.testing.assert_array_equal(res.Q, [[1.0]])
    res, _, _, _ = pkg.run(np.array([[0.0, 1.0], [1.0, 0.0]]), pkg.PipelineConfig(workers=2, b=4))
    np.testing.assert_allclose(res.lam, [-1.0, 1.0], atol=1e-15)
    assert orc.orthogonality(res.Q) < 4 * EPS


def test_six_spectra(G):
    # test_acceptance.py:34-50 at n=64 (the golden file stores the reference's matrices)
    for idx in range(6):
        a = G[f"spec{idx}_a"]
        res, _, _, _ = pkg.run(a, pkg.PipelineConfig(workers=2, b=8))
        lam_ref = G[f"spec{idx}_runlam"]
        np.testing.assert_allclose(res.lam, lam_ref, atol=10 * 64 * EPS * np.abs(lam_ref).max())
        assert orc.backward_error(a, res.Q, res.lam) <= 1e-15
        assert orc.orthogonality(res.Q) <= 1e-15


def test_planted_spectra_n1024():
    # test_acceptance.py:34-50 at the reference's size: planted spectra, 4 workers, b=32
    n = 1024
    rng = np.random.default_rng(1)
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    specs = {"Cluster0": np.r_[np.full(n - 1, 1e-2), 1e6], "Cluster1": np.r_[1e-2, np.full(n - 1, 1e6)],
             "Geometric": 1e6 * 1e8 ** (-np.arange(n) / (n - 1)),
             "Arithmetic": 1e6 * (1 - (1 - 1e-8) * np.arange(n) / (n - 1)),
             "Normal": rng.standard_normal(n), "Uniform": rng.uniform(-1, 1, n)}
    for name, lam in specs.items():
        a = (v * lam) @ v.T
        a = (a + a.T) / 2
        res, _, _, _ = pkg.run(a, pkg.PipelineConfig(workers=4, b=32))
        assert orc.backward_error(a, res.Q, res.lam) <= 1e-15, name
        assert orc.orthogonality(res.Q) <= 1e-15, name
        np.testing.assert_allclose(res.lam, np.sort(lam), atol=10 * n * EPS * np.abs(lam).max())


def test_fifty_random_matrices_vs_dense_solver():
    # test_acceptance.py:79-94
    rng = np.random.default_rng(0)
    worst = 0.0
    for _ in range(50):
        n = int(rng.integers(8, 65))
        workers = int(rng.integers(1, 5))
        b = int(rng.integers(2, 17))
        g = rng.standard_normal((n, n))
        a = (g + g.T) / 2
        res, _, _, _ = pkg.run(a, pkg.PipelineConfig(workers=min(workers, n), b=b))
        ref = np.linalg.eigvalsh(a)
        worst = max(worst, float(np.abs(res.lam - ref).max() / np.abs(ref).max()))
    assert worst <= 1e-12


def test_auto_skew():
    a = _sym(96, 16)
    res, events, ledger, counter, skew = pkg.run_auto_skew(a, pkg.PipelineConfig(workers=3, b=8))
    assert 0.0 <= skew <= 0.05
    assert orc.orthogonality(res.Q) <= 2 * EPS * 16


def test_stage_functions_match_reference_semantics():
    # per-stage API (sbr_reduce -> bc_reduce -> tridiag_eig -> back transforms), test_acceptance.py:66-73
    n, b = 96, 8
    a = pkg.SymmetricMatrix.from_dense(_sym(n, 2))
    band, factors = pkg.sbr_reduce(a, pkg.SbrConfig(b=b))
    t, u = pkg.bc_reduce(band)
    r = pkg.tridiag_eig(t, want_vectors=True)
    qs = pkg.sbr_back_accumulate(factors, (0, n))
    q_sb = pkg.bc_back_apply(u, np.ascontiguousarray(qs.T)).T
    q = pkg.final_gemm(q_sb, r.Q)
    assert orc.backward_error(a.data, q, r.lam) <= 1e-15
    rows = pkg.sbr_back_rows(factors, (10, 50))
    np.testing.assert_allclose(rows, qs[10:50], atol=1e-14)
    conv = pkg.bc_back_apply(u, np.eye(n), direction="conventional")
    reord = pkg.bc_back_apply(u, np.eye(n), direction="reordered")
    np.testing.assert_allclose(conv, reord.T, atol=1e-13)
    bands_o, _ = orc.sbr_reduce(a.data, b)
    np.testing.assert_allclose(band.bands, bands_o, atol=1e-12 * a.norm_f)


def test_stage_primitives_match_oracle():
    # core.py:258-306 / sbr.py:119-152 primitives on the DMMA GEMM
    rng = np.random.default_rng(3)
    m, k = 200, 8
    y = np.tril(rng.standard_normal((m, k)), -1)
    y[np.arange(k), np.arange(k)] = 1.0
    w = rng.standard_normal((m, k))
    panel = pkg.ReflectorPanel(W=w, Y=y, col_offset=0)
    c = rng.standard_normal((m, 17))
    for side, tr, want in (("left", False, c - w @ (y.T @ c)), ("left", True, c - y @ (w.T @ c))):
        got = pkg.apply_block_reflector(c.copy(), panel, side=side, transpose=tr)
        np.testing.assert_allclose(got, want, atol=1e-12)
    cr = rng.standard_normal((9, m))
    got = pkg.apply_block_reflector(cr.copy(), panel, side="right")
    np.testing.assert_allclose(got, cr - (cr @ w) @ y.T, atol=1e-12)
    a = rng.standard_normal((m, m))
    a = (a + a.T) / 2
    z = rng.standard_normal((m, k))
    got = pkg.sym_rank2k_update(a.copy(), y, z)
    np.testing.assert_array_equal(got, got.T)
    np.testing.assert_allclose(got, a - y @ z.T - z @ y.T, atol=1e-12)
    np.testing.assert_allclose(pkg.form_z(a, w, y), orc.form_z(a, w, y), atol=1e-11)


def test_row_accumulator_and_orders():
    n, b = 96, 8
    a = pkg.SymmetricMatrix.from_dense(_sym(n, 21))
    band, factors = pkg.sbr_reduce(a, pkg.SbrConfig(b=b))
    acc = pkg.RowAccumulator(n, (10, 60))
    for p in factors.panels:
        acc.apply_panel(p)
    np.testing.assert_allclose(acc.matrix(), pkg.sbr_back_rows(factors, (10, 60)), atol=1e-13)
    _, u = pkg.bc_reduce(band)
    for direction in ("reordered", "conventional"):
        u.validate_order(pkg.application_order(u, direction), direction)
    with pytest.raises(ValueError, match="dependency"):
        u.validate_order(pkg.application_order(u, "reordered")[::-1], "reordered")


def test_large_input_checked_on_device():
    """n > HOST_CHECK_MAX_N: the SymmetricMatrix check (core.py:75-84) runs on the device
    (pevd_asymmetry) and the host array is not transposed; C- and F-ordered inputs give the
    same eigenvalues, Q comes back in the reference's order per mode (pipeline.py:495, 503)."""
    from paper_2511_16174_b200.pipeline import HOST_CHECK_MAX_N
    n = HOST_CHECK_MAX_N + 100
    a = _sym(n, 77)
    res_c, _, _, _ = pkg.run(a, pkg.PipelineConfig(workers=1, b=32, order="pipelined"))
    assert res_c.Q.flags.c_contiguous
    res_f, _, _, _ = pkg.run(np.asfortranarray(a), pkg.PipelineConfig(workers=1, b=32,
                                                                       order="conventional"))
    assert res_f.Q.flags.f_contiguous
    lam_ref = np.linalg.eigvalsh(a)
    for r in (res_c, res_f):
        np.testing.assert_allclose(r.lam, lam_ref, atol=10 * n * EPS * np.abs(lam_ref).max())
    assert orc.backward_error(a, res_c.Q, res_c.lam) <= 1e-15
    assert orc.orthogonality(res_f.Q) <= 1e-15
    # conventional order with a C-ordered input: one native call (pevd_syevd_checked) that
    # uploads, checks, solves and streams Q back into a Fortran-ordered numpy array
    res_cc, _, _, _ = pkg.run(a, pkg.PipelineConfig(workers=1, b=32, order="conventional"))
    assert res_cc.Q.flags.f_contiguous
    np.testing.assert_allclose(res_cc.lam, res_f.lam, atol=1e-13 * np.abs(lam_ref).max())
    assert orc.backward_error(a, res_cc.Q, res_cc.lam) <= 1e-15
    bad = a.copy()
    bad[7, 3] += 1e-6
    for order in ("pipelined", "conventional"):
        with pytest.raises(ValueError, match="asymmetry"):
            pkg.run(bad, pkg.PipelineConfig(workers=1, b=32, order=order))


def test_device_asymmetry_kernel_matches_numpy():
    import ctypes
    import torch
    from paper_2511_16174_b200 import _lib
    L = _lib.load()
    for n in (1, 31, 33, 100, 1000):
        g = np.random.default_rng(n).standard_normal((n, n))
        d = torch.from_numpy(g.T.copy()).cuda()      # column-major g
        out = (ctypes.c_double * 2)()
        _lib.check(L.pevd_asymmetry(n, ctypes.c_void_p(d.data_ptr()), n, out, None), "asym")
        assert out[0] == np.abs(g - g.T).max()
        assert abs(out[1] - np.linalg.norm(g)) <= 1e-12 * np.linalg.norm(g)
