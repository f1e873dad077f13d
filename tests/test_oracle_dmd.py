"""Pins the oracle's cDMD small solve, modes, background and mask to closed forms
and special cases the paper fixes (Alg. 1; Eq. cDMDModes P:318-321;
Eq. DMDTerms; Eq. thres)."""

import numpy as np
import pytest

from oracle import cdmd as D
from oracle import sensing as S
from synth.scene import make_video


def _match(a, b):
    """max relative distance after greedy nearest matching of two eigenvalue sets."""
    a, b = list(a), list(b)
    worst = 0.0
    for x in a:
        j = int(np.argmin([abs(x - y) for y in b]))
        worst = max(worst, abs(x - b[j]) / max(abs(x), 1e-300))
        b.pop(j)
    return worst


def test_identity_sensing_reproduces_exact_dmd():
    # C = I (single pixel with p = n, a row permutation): cDMD == exact DMD
    # (§3: "The compressed DMD algorithm proceeds similarly to the standard DMD
    # algorithm ... until the computation of the DMD modes").
    # Exact DMD written independently: A^ = X' X^+  via the pseudoinverse;
    # its non-zero eigenvalues are the DMD eigenvalues and Phi are eigenvectors.
    rng = np.random.default_rng(0)
    n, m = 40, 13
    X = rng.integers(0, 256, size=(m, n), dtype=np.uint8)
    Xl = X[:-1].T.astype(np.float64)
    Xr = X[1:].T.astype(np.float64)
    Ahat = Xr @ np.linalg.pinv(Xl)
    ev = np.linalg.eigvals(Ahat)
    ev = ev[np.argsort(-np.abs(ev))][:m - 1]
    Y = S.sketch(X, S.SPIXEL, n, seed=3)
    model = D.fit(Y, k=m - 1, K=2)
    assert model["k_eff"] == m - 1
    assert _match(model["lam"], ev) < 1e-8
    Phi = D.modes(X, model["M"])
    for j in range(model["k_eff"]):
        r = Ahat @ Phi[:, j] - model["lam"][j] * Phi[:, j]
        assert np.linalg.norm(r) < 1e-8 * np.linalg.norm(Ahat) * np.linalg.norm(Phi[:, j])


def test_uint8_periodic_video_gives_roots_of_unity():
    # x_t = a + b1 cos(pi(t-1)/2) + b2 sin(pi(t-1)/2), integer-valued and exactly
    # 4-periodic: the DMD eigenvalues are exactly {1, i, -i}, omega = {0, +-i pi/2}
    # (Eq. omegaj, omega = log(lambda)/dt P:155).
    X = make_video(32, 24, 40, seed=9, noise=0.0, n_rects=0)
    Y = S.sketch(X, S.SPARSE, 50, seed=0)
    model = D.fit(Y, k=10, K=2)
    assert model["k_eff"] == 3
    assert _match(model["lam"], [1, 1j, -1j]) < 1e-10
    for w in (0.0, 0.5j * np.pi, -0.5j * np.pi):
        assert np.min(np.abs(model["omega"] - w)) < 1e-9
    # background = the video itself (exactly representable by the 3 modes)
    Phi = D.modes(X, model["M"])
    model3 = D.fit(Y, k=10, K=3)
    Phi3 = D.modes(X, model3["M"])
    L = D.background_dynamic(Phi3, model3)
    assert np.max(np.abs(L.T - X)) < 1e-8
    assert not D.mask(X, L, 0.5).any()
    assert Phi.shape == (768, 3)


def test_planted_exponentials_recovered():
    # fp64 planted modes {1, 0.98 e^{+-0.3i}}: eigenvalues to 1e-8
    rng = np.random.default_rng(1)
    n, m = 3000, 60
    lam = np.array([1.0, 0.98 * np.exp(0.3j), 0.98 * np.exp(-0.3j)])
    v0 = rng.standard_normal(n)
    v1 = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    V = np.stack([v0, v1, np.conj(v1)], 1)
    b = np.array([5.0, 2 + 1j, 2 - 1j])
    t = np.arange(m)
    Xf = (V * b) @ (lam[:, None] ** t[None, :])
    Xf = Xf.real                                   # (n, m)
    for kind in (S.GAUSSIAN, S.RADEMACHER):
        C = S.dense_C(kind, n, 40, seed=2).astype(np.float64)
        model = D.fit(C @ Xf, k=8, K=3)
        assert model["k_eff"] == 3
        assert _match(model["lam"], lam) < 1e-8


def test_static_video_background_is_the_frame():
    # a constant video: lambda = 1, background = the frame, empty mask
    rng = np.random.default_rng(2)
    frame = rng.integers(0, 256, size=500, dtype=np.uint8)
    X = np.tile(frame, (20, 1))
    Y = S.sketch(X, S.SPARSE, 30, seed=0, s=5.0)
    model = D.fit(Y, k=5, K=3)
    assert model["k_eff"] == 1
    assert abs(model["lam"][0] - 1) < 1e-12
    Phi = D.modes(X, model["M"])
    xs = D.background_static(Phi, model)
    assert np.max(np.abs(xs - frame)) < 1e-9
    Ld = D.background_dynamic(Phi, model)
    assert np.max(np.abs(Ld.T - X)) < 1e-9
    assert not D.mask(X, xs, 1e-3).any()


def test_doubling_sequence_lambda_two():
    # x_t = 2^(t-1) [1, 1] -> lambda = 2, through the identity sketch
    m = 8
    Yf = np.array([[2.0 ** t for t in range(m)]] * 2)
    model = D.fit(Yf, k=2, K=1)
    assert model["k_eff"] == 1 and abs(model["lam"][0] - 2) < 1e-12


def test_compressed_modes_are_sketched_full_modes():
    # Phi_Y = Y' V S^-1 W and Phi = X' V S^-1 W => Phi_Y = C Phi
    X = make_video(48, 32, 30, seed=4, noise=2.0, n_rects=1)
    n = X.shape[1]
    for kind in (S.SPARSE, S.RADEMACHER, S.SPIXEL):
        Y = S.sketch(X, kind, 120, seed=1, s=6.0)
        model = D.fit(Y, k=10, K=3)
        Phi = D.modes(X, model["M"])
        C = S.dense_C(kind, n, 120, seed=1, s=6.0).astype(np.float64)
        assert np.allclose(C @ Phi, model["PhiY"], rtol=1e-9, atol=1e-9 * np.abs(model["PhiY"]).max())


def test_dynamic_background_at_t1_equals_static():
    # "At time t = 1, equation (omegaj) reduces to x~_1 = sum_j b_j phi_j"
    X = make_video(40, 30, 25, seed=6, noise=2.0, n_rects=1)
    Y = S.sketch(X, S.SPARSE, 60, seed=0)
    model = D.fit(Y, k=8, K=4)
    Phi = D.modes(X, model["M"])
    Ld = D.background_dynamic(Phi, model, t0=0, nt=1)[:, 0]
    assert np.allclose(Ld, D.background_static(Phi, model), rtol=0, atol=1e-9)


def test_truncated_svd_reconstruction_and_atilde_similarity():
    # U S V* is the best rank-k approximation (Eckart-Young) and A~ is the
    # projection U* A^_Y U of A^_Y = Y' Y^+ 
    rng = np.random.default_rng(3)
    Yf = rng.standard_normal((50, 21))
    model = D.fit(Yf, k=20, K=2)
    Y, Yp = Yf[:, :-1], Yf[:, 1:]
    U, s, V = model["U"], model["sigma"], model["V"]
    assert np.allclose(U @ np.diag(s) @ V.T, Y, atol=1e-10)
    Ahat = Yp @ np.linalg.pinv(Y)
    assert np.allclose(U.T @ Ahat @ U, model["Atilde"], atol=1e-10)


def test_eigen_canonical_form():
    rng = np.random.default_rng(7)
    A = rng.standard_normal((9, 9))
    lam, W, pair = D.canonical_eig(A)
    assert np.allclose(A @ W, W * lam, atol=1e-10)
    assert np.all(np.diff(np.abs(lam)) <= 1e-12)
    for j in range(9):
        w = W[:, j]
        assert abs(np.linalg.norm(w) - 1) < 1e-12
        i = np.argmax(np.abs(w))
        assert abs(w[i].imag) < 1e-15 and w[i].real > 0
        if pair[j] == 1:
            assert lam[j].imag > 0 and lam[j + 1] == np.conj(lam[j]) and pair[j + 1] == -1
            assert np.array_equal(W[:, j + 1], np.conj(W[:, j]))
        if pair[j] == 0:
            assert lam[j].imag == 0


def test_fold_roundtrip():
    rng = np.random.default_rng(8)
    A = rng.standard_normal((6, 6))
    lam, W, pair = D.canonical_eig(A)
    F = D.fold(W, pair)
    for j in range(6):
        if pair[j] == 0:
            assert np.array_equal(F[:, j], W[:, j].real)
        elif pair[j] == 1:
            assert np.array_equal(F[:, j] + 1j * F[:, j + 1], W[:, j])


def test_mask_threshold_semantics():
    # Eq. thres: 1 iff |x_jt - xhat_j| > tau, strict (reading R16)
    X = np.array([[10, 20, 30, 40]], dtype=np.uint8)
    xh = np.array([10.0, 25.0, 30.0, 0.0])
    assert D.mask(X, xh, 5.0).tolist() == [[False, False, False, True]]
    assert D.mask(X, xh, 4.999).tolist() == [[False, True, False, True]]
    rng = np.random.default_rng(0)
    X = rng.integers(0, 256, size=(7, 100), dtype=np.uint8)
    L = rng.uniform(0, 255, size=(100, 7))
    prev = None
    for tau in [0.5, 5, 25, 60, 200]:
        mk = D.mask(X, L, tau)
        if prev is not None:
            assert np.all(mk <= prev)                  # monotone in tau
        prev = mk


def test_pack_unpack_roundtrip():
    rng = np.random.default_rng(0)
    for n in (1, 31, 32, 33, 100, 768):
        Mb = rng.random((5, n)) < 0.3
        Wd = D.pack_mask(Mb)
        assert Wd.shape == (5, (n + 31) // 32) and Wd.dtype == np.dtype("<u4")
        assert np.array_equal(D.unpack_mask(Wd, n), Mb)
        j = int(np.flatnonzero(Mb[0])[0]) if Mb[0].any() else None
        if j is not None:
            assert (int(Wd[0, j // 32]) >> (j % 32)) & 1 == 1


@pytest.mark.parametrize("kind", [S.SPIXEL, S.SPARSE, S.RADEMACHER, S.GAUSSIAN])
def test_whole_pipeline_detects_moving_object(kind):
    # quality sanity check (not a parity criterion): the object dominates the mask
    X = make_video(64, 48, 60, seed=11, noise=1.0, n_rects=1)
    res = D.cdmd(X, kind, p=400 if kind == S.SPIXEL else 200, k=12, K=6, tau=40.0)
    truth = X >= 250
    mk = res["mask"]
    tp = np.sum(mk & truth)
    assert tp / max(1, mk.sum()) > 0.5 and tp / max(1, truth.sum()) > 0.5
