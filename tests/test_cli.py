"""The command-line front end and EVD1 files, mirroring the reference's tests/test_cli.py and
tests/test_evdio.py.  `gen`, the file format and the argument errors run on CPU; `solve` runs the
EVD on the GPU (marked)."""
import json
import struct

import numpy as np
import pytest

from paper_2511_16174_b200 import matgen
from paper_2511_16174_b200.cli import EXIT_OK, EXIT_USAGE, EXIT_VERIFY, main
from paper_2511_16174_b200.evdio import (MAGIC, read_matrix, read_vector, write_rect,
                                         write_square, write_vector)

G = np.load("tests/golden/golden.npz")


def _gen(tmp_path, n=32, dist="uniform", seed=3):
    out = tmp_path / "gen"
    assert main(["gen", "--n", str(n), "--dist", dist, "--seed", str(seed),
                 "--out", str(out)]) == EXIT_OK
    return out / "matrix.evd1"


# ---------------------------------------------------------------- EVD1 files (test_evdio.py)
def test_square_and_rect_round_trip(tmp_path):
    a = np.asfortranarray(np.arange(12.0).reshape(3, 4))
    write_rect(tmp_path / "r.evd1", a)
    np.testing.assert_array_equal(read_matrix(tmp_path / "r.evd1"), a)
    s = np.random.default_rng(0).standard_normal((5, 5))
    write_square(tmp_path / "s.evd1", s)
    raw = (tmp_path / "s.evd1").read_bytes()
    assert raw[:4] == MAGIC and struct.unpack_from("<Q", raw, 4)[0] == 5
    assert len(raw) == 12 + 8 * 25
    np.testing.assert_array_equal(read_matrix(tmp_path / "s.evd1"), s)
    v = np.linspace(-1, 1, 7)
    write_vector(tmp_path / "v.evd1", v)
    np.testing.assert_array_equal(read_vector(tmp_path / "v.evd1"), v)


def test_bad_files(tmp_path):
    (tmp_path / "x.evd1").write_bytes(b"NOPE" + bytes(20))
    with pytest.raises(ValueError, match="not an EVD1"):
        read_matrix(tmp_path / "x.evd1")
    (tmp_path / "t.evd1").write_bytes(MAGIC + b"\x01")
    with pytest.raises(ValueError, match="truncated"):
        read_matrix(tmp_path / "t.evd1")
    (tmp_path / "h.evd1").write_bytes(MAGIC + struct.pack("<QQ", 3, 3) + bytes(8))
    with pytest.raises(ValueError, match="inconsistent"):
        read_matrix(tmp_path / "h.evd1")
    with pytest.raises(ValueError):
        write_square(tmp_path / "n.evd1", np.zeros((2, 3)))
    write_rect(tmp_path / "m.evd1", np.zeros((3, 2)))
    with pytest.raises(ValueError, match="column vector"):
        read_vector(tmp_path / "m.evd1")


# ---------------------------------------------------------------- gen (host, reference-exact)
@pytest.mark.parametrize("idx", range(6))
def test_host_generator_matches_reference(idx):
    kind = str(G[f"spec{idx}_kind"])
    a, lam = matgen.generate_host(matgen.SpectrumSpec(kind, 64, seed=1))
    np.testing.assert_array_equal(a, G[f"spec{idx}_a"])
    np.testing.assert_array_equal(lam, G[f"spec{idx}_lam"])


def test_gen_writes_matrix_and_sidecar(tmp_path, capsys):
    mpath = _gen(tmp_path)
    a = read_matrix(mpath)
    assert a.shape == (32, 32)
    np.testing.assert_array_equal(a, a.T)
    lam = read_vector(tmp_path / "gen" / "matrix.spectrum.evd1")
    assert np.all(np.diff(lam) >= 0.0)
    np.testing.assert_allclose(np.linalg.eigvalsh(a), lam, atol=1e-13)
    assert "matrix.evd1" in capsys.readouterr().out


def test_gen_is_deterministic(tmp_path):
    m1 = _gen(tmp_path / "a", seed=5)
    m2 = _gen(tmp_path / "b", seed=5)
    assert m1.read_bytes() == m2.read_bytes()
    assert m1.read_bytes() != _gen(tmp_path / "c", seed=6).read_bytes()


def test_usage_errors(tmp_path, capsys):
    assert main(["gen", "--n", "8", "--dist", "bogus", "--out", str(tmp_path)]) == EXIT_USAGE
    assert "unknown spectrum kind" in capsys.readouterr().err
    mpath = _gen(tmp_path, n=16)
    assert main(["solve", str(mpath), "--n", "16", "--out", str(tmp_path / "x")]) == EXIT_USAGE
    assert "not both" in capsys.readouterr().err
    assert main(["solve", "--n", "16", "--out", str(tmp_path / "x")]) == EXIT_USAGE
    assert "required" in capsys.readouterr().err
    assert main(["solve", str(tmp_path / "missing.evd1"),
                 "--out", str(tmp_path / "x")]) == EXIT_USAGE
    assert main(["simulate", "--n", "64", "--model", str(tmp_path / "nope.json")]) == EXIT_USAGE
    assert "malformed cost model" in capsys.readouterr().err


def test_simulate(tmp_path, capsys):
    """cli.py simulate (reference cli.py:209-231): both orders priced, trace written."""
    from paper_2511_16174_b200.messaging import TraceLog
    from paper_2511_16174_b200.schedule import validate_trace
    trace = tmp_path / "sim.ndjson"
    for model in ("calibrated", "b200", "unit"):
        assert main(["simulate", "--n", "4096", "--workers", "4", "--model", model,
                     "--trace", str(trace)]) == 0
        out = capsys.readouterr().out
        assert "pipelined  makespan" in out and "ratio" in out
        validate_trace(TraceLog.from_ndjson(trace), 4)

# ---------------------------------------------------------------- solve / verify (GPU)
@pytest.mark.gpu
def test_solve_from_file_and_verify(tmp_path, capsys):
    from paper_2511_16174_b200.messaging import TraceLog
    mpath = _gen(tmp_path, n=48)
    out = tmp_path / "run"
    assert main(["solve", str(mpath), "--workers", "2", "--band", "8",
                 "--out", str(out)]) == EXIT_OK
    lam = read_vector(out / "lambda.evd1")
    np.testing.assert_allclose(lam, np.linalg.eigvalsh(read_matrix(mpath)), atol=1e-12)
    assert read_matrix(out / "Q.evd1").shape == (48, 48)
    assert (out / "ledger.csv").read_text().startswith("src,dst,stage,words")
    assert (out / "flops.csv").read_text().startswith("stage,multiply_adds")
    assert len(TraceLog.from_ndjson(out / "trace.ndjson")) > 0
    manifest = json.loads((out / "manifest.json").read_text())
    assert manifest["command"] == "solve" and manifest["config"]["n"] == 48
    assert manifest["config"]["workers"] == 2 and manifest["config"]["matrix"] == str(mpath)
    assert manifest["metrics"]["accuracy"]["bound_ok"] is True
    assert manifest["metrics"]["comm_total_words"] > 0
    capsys.readouterr()
    assert main(["verify", str(mpath), str(out)]) == EXIT_OK
    report = json.loads(capsys.readouterr().out)
    assert report["bound_ok"] is True and report["backward"] <= 1e-15


@pytest.mark.gpu
def test_solve_inline_and_values_only(tmp_path, capsys):
    out = tmp_path / "run"
    assert main(["solve", "--n", "40", "--dist", "geometric", "--cond", "1e4", "--workers", "3",
                 "--band", "4", "--order", "conventional", "--out", str(out)]) == EXIT_OK
    manifest = json.loads((out / "manifest.json").read_text())
    assert manifest["config"]["matrix"] is None and manifest["config"]["dist"] == "geometric"
    mpath = _gen(tmp_path, n=32)
    vals = tmp_path / "vals"
    assert main(["solve", str(mpath), "--vectors", "off", "--band", "8",
                 "--out", str(vals)]) == EXIT_OK
    assert not (vals / "Q.evd1").exists()
    capsys.readouterr()
    assert main(["verify", str(mpath), str(vals)]) == EXIT_OK
    assert json.loads(capsys.readouterr().out)["mode"] == "eigenvalues"


@pytest.mark.gpu
def test_verify_catches_corruption(tmp_path, capsys):
    mpath = _gen(tmp_path, n=24)
    out = tmp_path / "run"
    assert main(["solve", str(mpath), "--band", "4", "--out", str(out)]) == EXIT_OK
    q = read_matrix(out / "Q.evd1")
    q[3, 3] += 1e-3
    write_square(out / "Q.evd1", q)
    capsys.readouterr()
    assert main(["verify", str(mpath), str(out)]) == EXIT_VERIFY
    assert json.loads(capsys.readouterr().out)["bound_ok"] is False


@pytest.mark.gpu
def test_solve_device_generated(tmp_path, capsys):
    out = tmp_path / "dev"
    assert main(["solve", "--n", "2048", "--dist", "normal", "--device-gen", "--order",
                 "conventional", "--out", str(out)]) == EXIT_OK
    manifest = json.loads((out / "manifest.json").read_text())
    lam = read_vector(out / "lambda.evd1")
    ref = matgen.eigen_spectrum(matgen.SpectrumSpec("normal", 2048))
    np.testing.assert_allclose(lam, ref, atol=10 * 2048 * 2.3e-16 * np.abs(ref).max())
    assert manifest["metrics"]["accuracy"]["bound_ok"] is True
