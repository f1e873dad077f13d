"""Pins the oracle's OMP (Remark 3) against exhaustive
search and closed forms."""

import itertools

import numpy as np

from oracle.cdmd import omp


def _exhaustive(D, y, K):
    best, arg = np.inf, None
    for S in itertools.combinations(range(D.shape[1]), K):
        b = np.linalg.lstsq(D[:, S], y, rcond=None)[0]
        r = np.linalg.norm(y - D[:, S] @ b)
        if r < best - 1e-12:
            best, arg = r, S
    return set(arg), best


def test_identity_dictionary():
    # D = I: OMP picks the K largest |y_i| and beta = y on them
    y = np.array([0.5, -3.0, 2.0, 0.1, -1.0])
    S, b = omp(np.eye(5), y, 3)
    assert S == [1, 2, 4]
    assert np.allclose(b, y[S])


def test_k1_equals_exhaustive_search():
    rng = np.random.default_rng(0)
    for _ in range(50):
        D = rng.standard_normal((12, 7)) + 1j * rng.standard_normal((12, 7))
        y = rng.standard_normal(12)
        S, b = omp(D, y, 1)
        Se, re = _exhaustive(D, y, 1)
        assert set(S) == Se
        assert abs(np.linalg.norm(y - D[:, S] @ b) - re) < 1e-10


def test_planted_sparse_supports_recovered():
    rng = np.random.default_rng(1)
    for K in (1, 2, 3):
        for _ in range(40):
            # Tropp (2004): OMP recovers every K-sparse representation when
            # K < (1 + 1/mu) / 2, mu the mutual coherence of the unit columns
            D = rng.standard_normal((400, 10))
            D /= np.linalg.norm(D, axis=0)
            G = np.abs(D.T @ D) - np.eye(10)
            assert K < (1 + 1 / G.max()) / 2
            T = sorted(rng.choice(10, K, replace=False).tolist())
            c = rng.uniform(1, 2, K) * rng.choice([-1, 1], K)
            y = D[:, T] @ c
            S, b = omp(D, y, K)
            assert sorted(S) == T
            assert set(S) == _exhaustive(D, y, K)[0]
            assert np.allclose(np.asarray(b).real[np.argsort(S)], c, atol=1e-10)


def test_full_k_is_least_squares():
    rng = np.random.default_rng(2)
    D = rng.standard_normal((30, 6)) + 1j * rng.standard_normal((30, 6))
    y = rng.standard_normal(30)
    S, b = omp(D, y, 6)
    assert sorted(S) == list(range(6))
    full = np.linalg.lstsq(D, y, rcond=None)[0]
    r1 = np.linalg.norm(y - D[:, S] @ b)
    r2 = np.linalg.norm(y - D @ full)
    assert abs(r1 - r2) < 1e-10


def test_residual_orthogonal_and_monotone():
    rng = np.random.default_rng(3)
    D = rng.standard_normal((25, 9)) + 1j * rng.standard_normal((25, 9))
    y = rng.standard_normal(25)
    prev = np.inf
    for K in range(1, 7):
        S, b = omp(D, y, K)
        r = y - D[:, S] @ b
        assert np.abs(D[:, S].conj().T @ r).max() < 1e-10
        assert np.linalg.norm(r) <= prev + 1e-12
        prev = np.linalg.norm(r)


def test_conjugate_pair_tie_takes_lower_index():
    # for a real target, the two members of a conjugate pair of columns have
    # exactly equal correlation; reading R13 takes the lower index
    rng = np.random.default_rng(4)
    v = rng.standard_normal(20) + 1j * rng.standard_normal(20)
    w = rng.standard_normal(20)
    D = np.stack([w, v, np.conj(v)], 1)
    y = 5 * v.real + 0.01 * w
    S, _ = omp(D, y, 1)
    assert S == [1]


def test_early_stop_on_exact_fit():
    D = np.eye(4)
    y = np.array([1.0, 0, 0, 0])
    S, b = omp(D, y, 3)
    assert S == [0] and np.allclose(b, [1.0])
