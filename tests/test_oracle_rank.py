"""Pins for the Gavish-Donoho automatic target rank (Remark 2; the paper's
evaluation settings): oracle.cdmd.optimal_rank and fit(rank="gd")."""

import numpy as np
import pytest

from oracle import cdmd as OD


def test_omega_cubic_values():
    # the cubic of the cited unknown-noise rule at the square (beta = 1) and thin limits
    assert OD.omega_beta(1.0) == pytest.approx(2.86, abs=1e-12)
    assert OD.omega_beta(0.0) == pytest.approx(1.43, abs=1e-12)
    b = 0.25
    assert OD.omega_beta(b) == pytest.approx(0.56 * b**3 - 0.95 * b**2 + 1.82 * b + 1.43, abs=1e-15)


def test_one_dominant_value():
    assert OD.optimal_rank([10.0, 1e-12, 1e-13], 100, 99) == 1


def test_at_least_one_and_errors():
    assert OD.optimal_rank([1.0, 1.0, 1.0], 50, 50) == 1      # nothing above 2.86 x median
    with pytest.raises(ValueError):
        OD.optimal_rank([], 3, 3)


def test_recovers_planted_rank_under_noise():
    """rank-5 signal + i.i.d. noise at SNR 1e3, 200 x 200: rank 5 in >= 19 of 20 seeds."""
    hits = 0
    for seed in range(20):
        rng = np.random.default_rng(seed)
        n, r = 200, 5
        A = (rng.standard_normal((n, r)) * np.linspace(30, 10, r)) @ rng.standard_normal((r, n)) / np.sqrt(n)
        sr = np.linalg.svd(A, compute_uv=False)[r - 1]
        N = rng.standard_normal((n, n)) * (sr / 1e3) / np.sqrt(n)
        hits += OD.optimal_rank(np.linalg.svd(A + N, compute_uv=False), n, n) == r
    assert hits >= 19


def test_pure_noise_is_rank_one():
    """Marchenko-Pastur bulk lies below omega(beta) median: i.i.d. noise gives the floor of 1."""
    for seed in range(5):
        rng = np.random.default_rng(100 + seed)
        s = np.linalg.svd(rng.standard_normal((300, 120)), compute_uv=False)
        assert OD.optimal_rank(s, 300, 120) == 1


def test_fit_gd_picks_planted_rank():
    """Sketch of 4 real exponentials (2 real + 1 conjugate pair of DMD modes) plus small
    noise: fit(rank='gd', k=20) keeps exactly 4 singular values; with rank='fixed' and
    k = 4 the two fits coincide."""
    rng = np.random.default_rng(7)
    p, m = 120, 60
    t = np.arange(m)
    lam = [0.99, 0.9, 0.97 * np.exp(0.3j), 0.97 * np.exp(-0.3j)]
    modes = rng.standard_normal((p, 2)), (rng.standard_normal(p) + 1j * rng.standard_normal(p))
    Y = np.outer(modes[0][:, 0], lam[0] ** t) + np.outer(modes[0][:, 1], lam[1] ** t)
    Y = Y + 2 * np.real(np.outer(modes[1], lam[2] ** t))
    Y = Y + 1e-6 * rng.standard_normal((p, m))
    g = OD.fit(Y, 20, 2, rank="gd")
    f = OD.fit(Y, 4, 2)
    assert g["k_eff"] == 4
    np.testing.assert_allclose(np.sort_complex(g["lam"]), np.sort_complex(f["lam"]), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(np.sort(np.abs(g["lam"])), np.sort(np.abs(np.array(lam))), rtol=1e-5)
