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


def _mp_density(beta):
    """Marchenko-Pastur density of the squared singular values of an i.i.d. noise matrix
    with aspect ratio beta and unit entry variance (scaled by the long side)."""
    lo, hi = (1 - np.sqrt(beta)) ** 2, (1 + np.sqrt(beta)) ** 2
    return lo, hi, lambda x: np.sqrt(max((hi - x) * (x - lo), 0.0)) / (2 * np.pi * beta * x)


def _mp_median(beta):
    from scipy import integrate, optimize
    lo, hi, f = _mp_density(beta)
    return optimize.brentq(lambda mu: integrate.quad(f, lo, mu, limit=200)[0] - 0.5, lo + 1e-12, hi)


def _lambda_star(beta):
    """Gavish-Donoho optimal hard threshold for KNOWN noise level, in units of sqrt(n) sigma."""
    return np.sqrt(2 * (beta + 1) + 8 * beta / ((beta + 1) + np.sqrt(beta * beta + 14 * beta + 1)))


def test_mp_density_is_a_distribution():
    # sanity of the numerical Marchenko-Pastur law used below: total mass 1, mean 1
    from scipy import integrate
    for beta in (0.1, 0.5, 1.0):
        lo, hi, f = _mp_density(beta)
        assert integrate.quad(f, lo, hi, limit=200)[0] == pytest.approx(1.0, abs=1e-7)
        assert integrate.quad(lambda x: x * f(x), lo, hi, limit=200)[0] == pytest.approx(1.0, abs=1e-7)


def test_omega_cubic_matches_the_exact_unknown_noise_coefficient():
    """Remark 2 / evaluation settings use the unknown-noise rule
    tau = omega(beta) median(sigma).  Its exact coefficient is
    omega(beta) = lambda*(beta) / sqrt(mu_beta), mu_beta the Marchenko-Pastur median
    (Gavish & Donoho 2014); the cubic 0.56 b^3 - 0.95 b^2 + 1.82 b + 1.43 is their fit
    to it.  Pinned against the exact value within 1e-2 for beta in [0.05, 1] (measured
    worst 5.7e-3 at beta = 0.1): a wrong sign or coefficient of any term moves it by
    more (e.g. +0.95 b^2 gives 4.76 at beta = 1)."""
    for beta in (0.05, 0.1, 0.25, 0.5, 0.75, 1.0):
        exact = _lambda_star(beta) / np.sqrt(_mp_median(beta))
        assert abs(OD.omega_beta(beta) - exact) <= 1e-2, (beta, OD.omega_beta(beta), exact)
    # the two ingredients pinned on their own: lambda*(1) = 4 / sqrt(3) (closed form), and
    # mu_beta against the empirical median of the squared singular values of an i.i.d.
    # N(0, 1/n) matrix (Monte Carlo, 2000 x 2000 and 500 x 2000)
    assert _lambda_star(1.0) == pytest.approx(4 / np.sqrt(3), abs=1e-12)
    rng = np.random.default_rng(0)
    for rows, beta in ((2000, 1.0), (500, 0.25)):
        Z = rng.standard_normal((rows, 2000)) / np.sqrt(2000)
        emp = np.median(np.linalg.svd(Z, compute_uv=False) ** 2)
        assert _mp_median(beta) == pytest.approx(emp, abs=4e-3), (beta, emp)


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
