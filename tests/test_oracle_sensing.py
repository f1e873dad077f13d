"""Pins the oracle's measurement matrices and sketch Y = C X.

Each pin checks something the paper or the mathematics fixes, not the oracle's
own formula: distributions (binomial / geometric / moment confidence bounds),
without-replacement sampling (a permutation at p = n), the energy identities
E||C x||^2, exact integer brute force against a materialised C, slab
additivity, and rank preservation.
"""

import math
import statistics

import numpy as np
import pytest

from oracle import sensing as S
from synth.scene import make_video


@pytest.mark.parametrize("n", [1, 2, 7, 64, 100, 768, 1000, 4097])
def test_spixel_p_equals_n_is_permutation(n):
    # "draws p random rows (without replacement)": at p = n all rows.
    rows = S.spixel_rows(n, n, seed=123)
    assert sorted(rows.tolist()) == list(range(n))


def test_spixel_rows_distinct_and_uniform():
    n, p, trials = 200, 20, 400
    counts = np.zeros(n)
    for sd in range(trials):
        r = S.spixel_rows(n, p, seed=sd)
        assert len(set(r.tolist())) == p and r.min() >= 0 and r.max() < n
        counts[r] += 1
    # each pixel included w.p. p/n; chi-square over n cells with n-1 dof
    e = trials * p / n
    chi2 = ((counts - e) ** 2 / e).sum()
    assert chi2 < (n - 1) + 6 * math.sqrt(2 * (n - 1))


def test_sparse_entry_distribution():
    # c_ij = +1 w.p. 1/(2s), -1 w.p. 1/(2s), 0 w.p. 1 - 1/s
    n, p, s = 5000, 200, 25.0
    C = S.dense_C(S.SPARSE, n, p, seed=7, s=s)
    N = n * p
    nz = np.count_nonzero(C)
    mu, sd = N / s, math.sqrt(N / s * (1 - 1 / s))
    assert abs(nz - mu) < 5 * sd
    pos = np.count_nonzero(C == 1)
    assert abs(pos - nz / 2) < 5 * math.sqrt(nz / 4)
    assert set(np.unique(C).tolist()) <= {-1, 0, 1}


def test_sparse_gaps_are_geometric():
    # i.i.d. Bernoulli(1/s) entries <=> gaps between non-zeros ~ Geometric(1/s)
    n, s = 200000, 40.0
    rows = S.sparse_rows(n, 8, s, seed=3)
    gaps = np.concatenate([np.diff(np.concatenate([[-1], pos])) - 1 for pos, _ in rows])
    q = 1 / s
    for k in (0, 10, 40, 100):
        emp = np.mean(gaps >= k)
        th = (1 - q) ** k
        assert abs(emp - th) < 5 * math.sqrt(th * (1 - th) / len(gaps)) + 1e-3


def test_sparse_default_s_is_n_over_ln_n():
    # s = n / log(n): about ln(n) non-zeros per row
    n, p = 2073600, 2000
    assert abs(S.default_s(n) - 142566.0) < 1.0
    rows = S.sparse_rows(n, p, S.default_s(n), seed=0)
    nnz = sum(len(r[0]) for r in rows)
    mu = p * math.log(n)
    assert abs(nnz - mu) < 5 * math.sqrt(mu)


def test_rademacher_entries_balanced_and_pairwise_uncorrelated():
    C = S.dense_C(S.RADEMACHER, 4096, 64, seed=11).astype(np.float64)
    assert set(np.unique(C).tolist()) == {-1.0, 1.0}
    N = C.size
    assert abs(C.sum()) < 5 * math.sqrt(N)
    G = C @ C.T / C.shape[1]          # rows nearly orthogonal: off-diagonal ~ N(0, 1/n)
    off = G[~np.eye(64, dtype=bool)]
    assert np.abs(off).max() < 6 / math.sqrt(4096)
    assert np.allclose(np.diag(G), 1.0)


def test_gaussian_table_against_independent_inverse_cdf():
    # N(0,1) entries rounded to bf16 (reading R7): compare with the
    # inverse CDF of Python's statistics module (a different implementation
    # than scipy.special.ndtri used by the oracle), rounded with float math.
    T = S.gaussian_table()
    nd = statistics.NormalDist()
    for j in [0, 1, 2, 17, 1000, 9999, 32767, 32768, 40000, 65534, 65535]:
        x = nd.inv_cdf((j + 0.5) / 65536)
        m, e = math.frexp(x)
        want = math.ldexp(round(m * 256), e - 8)   # round(): ties to even
        assert T[j] == want
    assert np.all(np.diff(T) >= 0)
    assert np.array_equal(T[::-1], -T)             # symmetric
    assert T[0] == -4.3125 and T[-1] == 4.3125
    assert abs(T.var() - 1.0) < 2e-5 and T.mean() == 0.0
    assert len(np.unique(T)) == 2680


def test_gaussian_entries_moments():
    C = S.dense_C(S.GAUSSIAN, 8192, 32, seed=5)
    N = C.size
    assert abs(C.mean()) < 5 / math.sqrt(N)
    assert abs(C.var() - 1.0) < 5 * math.sqrt(2.0 / N)
    # bf16-valued: 8 significant bits
    m, e = np.frexp(C[C != 0])
    assert np.all(np.ldexp(m, 8) == np.round(np.ldexp(m, 8)))


@pytest.mark.parametrize("kind", [S.SPIXEL, S.SPARSE])
def test_gather_sketch_equals_dense_brute_force(kind):
    # exact integer C D with C materialised from the same definition; the
    # sketch itself never materialises C (row gather / signed gather-sum).
    n, m, p = 700, 9, 60
    X = np.random.default_rng(0).integers(0, 256, size=(m, n), dtype=np.uint8)
    C = S.dense_C(kind, n, p, seed=42, s=9.0)
    Y = S.sketch(X, kind, p, seed=42, s=9.0)
    assert Y.dtype == np.int64
    assert np.array_equal(Y, C @ X.T.astype(np.int64))


def test_identity_video_returns_C():
    # frames = unit pixel vectors (D = I_n): Y = C exactly, for all four kinds
    n, p = 300, 40
    X = np.eye(n, dtype=np.uint8)
    for kind in (S.SPIXEL, S.SPARSE, S.RADEMACHER, S.GAUSSIAN):
        Y = S.sketch(X, kind, p, seed=9, s=5.0)
        C = S.dense_C(kind, n, p, seed=9, s=5.0)
        assert np.array_equal(Y, C)


@pytest.mark.parametrize("kind", [S.SPIXEL, S.SPARSE, S.RADEMACHER, S.GAUSSIAN])
def test_slabs_sum_to_full_sketch(kind):
    # columns of C are indexed by the global pixel index
    n, m, p = 1024, 6, 33
    X = np.random.default_rng(1).integers(0, 256, size=(m, n), dtype=np.uint8)
    full = S.sketch(X, kind, p, seed=5)
    parts = sum(S.sketch(X[:, a:b], kind, p, seed=5, n_total=n, pix0=a)
                for a, b in [(0, 256), (256, 640), (640, 1024)])
    if kind == S.GAUSSIAN:
        assert np.allclose(parts, full, rtol=1e-12, atol=1e-9)
    else:
        assert np.array_equal(parts, full)


def test_energy_identities():
    # E||C x||^2 = p ||x||^2 / s (sparse), p ||x||^2 (Rademacher),
    # (p/n) ||x||^2 (single pixel), p var(T) ||x||^2 (Gaussian)
    n, p, trials = 512, 16, 60
    x = np.random.default_rng(2).integers(0, 256, size=(1, n)).astype(np.uint8)
    e = float((x.astype(np.float64) ** 2).sum())
    s = 8.0
    want = {S.SPARSE: p * e / s, S.RADEMACHER: p * e, S.SPIXEL: p * e / n,
            S.GAUSSIAN: p * e * S.gaussian_table().var()}
    for kind, w in want.items():
        vals = [float((S.sketch(x, kind, p, seed=sd, s=s).astype(np.float64) ** 2).sum())
                for sd in range(trials)]
        mean, sem = np.mean(vals), np.std(vals) / math.sqrt(trials)
        assert abs(mean - w) < 5 * sem + 1e-9 * w, (kind, mean, w, sem)


@pytest.mark.parametrize("kind", [S.SPARSE, S.RADEMACHER, S.GAUSSIAN])
def test_rank_preserved(kind):
    # noiseless rank-r video, p >= 2r: rank(Y) = r (SPEC sensing invariants)
    rng = np.random.default_rng(4)
    n, m, r = 2000, 30, 4
    A = rng.integers(0, 8, size=(n, r)) @ rng.integers(0, 8, size=(r, m))
    X = np.clip(A, 0, 255).astype(np.uint8).T
    Y = S.sketch(X, kind, 3 * r, seed=1, s=4.0).astype(np.float64)
    sv = np.linalg.svd(Y, compute_uv=False)
    assert np.sum(sv > 1e-8 * sv[0]) == np.linalg.matrix_rank(X.astype(np.float64))


def test_periodic_scene_is_exact():
    # the synthetic generator's noiseless, object-free video is exactly 4-periodic
    X = make_video(32, 24, 12, seed=5, noise=0.0, n_rects=0)
    assert np.array_equal(X[:4], X[4:8]) and np.array_equal(X[:4], X[8:12])
