"""Host side of the planted-spectrum generator (paper_2511_16174_b200/matgen.py).

The six spectrum families are pinned against the reference's own eigen_spectrum output
(tests/golden/golden.npz, spec{i}_lam: matgen.generate(SpectrumSpec(kind, 64, seed=1)) of the
real reference), and the compact-WY T of the Householder basis is checked against the explicit
product of the reflectors.
"""
import numpy as np
import pytest

from paper_2511_16174_b200 import matgen

G = np.load("tests/golden/golden.npz")


@pytest.mark.parametrize("idx", range(6))
def test_spectrum_matches_reference(idx):
    kind = str(G[f"spec{idx}_kind"])
    lam = matgen.eigen_spectrum(matgen.SpectrumSpec(kind, 64, seed=1))
    np.testing.assert_array_equal(lam, G[f"spec{idx}_lam"])


def test_kind_lookup_and_validation():
    assert matgen.canonical_kind("geometric") == "Geometric"
    with pytest.raises(ValueError):
        matgen.canonical_kind("nope")
    with pytest.raises(ValueError):
        matgen.SpectrumSpec("Normal", 8, cond=0.5)
    with pytest.raises(ValueError):
        matgen.SpectrumSpec("Normal", 8, lambda_max=-1.0)
    with pytest.raises(ValueError):
        matgen.eigen_spectrum(matgen.SpectrumSpec("Normal", 1))


def test_householder_t_is_the_product():
    rng = np.random.default_rng(5)
    n, k = 40, 7
    Y = rng.standard_normal((n, k))
    T = matgen.householder_t(Y.T @ Y)
    Q = np.eye(n)
    for i in range(k):
        y = Y[:, i]
        Q = Q @ (np.eye(n) - 2.0 / (y @ y) * np.outer(y, y))
    np.testing.assert_allclose(np.eye(n) - Y @ T @ Y.T, Q, atol=1e-13)
    np.testing.assert_allclose(Q.T @ Q, np.eye(n), atol=1e-13)
