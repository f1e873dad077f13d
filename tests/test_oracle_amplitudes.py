"""Pins for oracle.cdmd.amplitudes: b = lstsq(Phi, x_1), Alg. 1 step 9."""

import numpy as np

from oracle import cdmd as D
from oracle import sensing as S
from synth.scene import make_video


def _frames(x1, m=3):
    return np.tile(np.asarray(x1, dtype=np.uint8), (m, 1))


def test_planted_integer_combination_recovered():
    # x_1 = a + 2 Re((1 - i)(u + i v)) = a + 2u + 2v exactly, so with the modes
    # [a, u + iv, u - iv] the unique least-squares solution is b = [1, 1 - i, 1 + i].
    rng = np.random.default_rng(3)
    n = 400
    a = rng.integers(0, 60, n).astype(np.float64)
    u = rng.integers(0, 40, n).astype(np.float64)
    v = rng.integers(0, 40, n).astype(np.float64)
    x1 = a + 2 * u + 2 * v
    Phi = np.stack([a, u + 1j * v, u - 1j * v], 1)
    b = D.amplitudes(_frames(x1), Phi)
    assert np.max(np.abs(b - np.array([1, 1 - 1j, 1 + 1j]))) < 1e-10


def test_orthonormal_modes_give_the_projection():
    # orthonormal columns: lstsq reduces to b = Phi^H x_1 (x_1 need not lie in the span)
    rng = np.random.default_rng(4)
    n, k = 300, 7
    Q, _ = np.linalg.qr(rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k)))
    x1 = rng.integers(0, 256, n)
    b = D.amplitudes(_frames(x1), Q)
    assert np.max(np.abs(b - Q.conj().T @ x1)) < 1e-9 * np.linalg.norm(x1)


def test_residual_orthogonal_to_the_modes_and_minimal():
    rng = np.random.default_rng(5)
    n, k = 500, 9
    Phi = rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k))
    x1 = rng.integers(0, 256, n).astype(np.float64)
    b = D.amplitudes(_frames(x1), Phi)
    r = x1 - Phi @ b
    assert np.linalg.norm(Phi.conj().T @ r) < 1e-9 * np.linalg.norm(Phi) * np.linalg.norm(x1)
    for _ in range(5):
        d = 1e-3 * (rng.standard_normal(k) + 1j * rng.standard_normal(k))
        assert np.linalg.norm(x1 - Phi @ (b + d)) > np.linalg.norm(r)


def test_periodic_video_amplitudes_reconstruct_every_frame():
    # the exactly 4-periodic uint8 video (lambda = 1, +-i): the full-state amplitudes
    # reproduce x_1 and, through lambda^(t-1), every frame (Eq. DMDTerms
    # with b from step 9 instead of OMP).
    X = make_video(32, 24, 40, seed=9, noise=0.0, n_rects=0)
    model = D.fit(S.sketch(X, S.SPARSE, 50, seed=0), k=10, K=2)
    Phi = D.modes(X, model["M"])
    b = D.amplitudes(X, Phi)
    assert np.max(np.abs((Phi @ b).real - X[0])) < 1e-8
    t = np.arange(X.shape[0])
    L = (Phi @ (b[:, None] * model["lam"][:, None] ** t[None, :])).real
    assert np.max(np.abs(L.T - X)) < 1e-7
    # conjugate members of a pair get conjugate amplitudes (x_1 is real)
    for j in np.nonzero(model["pair"] == 1)[0]:
        assert abs(b[j + 1] - np.conj(b[j])) < 1e-9 * np.max(np.abs(b))
