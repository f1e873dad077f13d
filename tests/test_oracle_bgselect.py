"""Pins the oracle's frequency-based background selection (the background is
modelled by the modes with |omega_p| ~ 0; selection by |omega| < eps, amplitudes by
least squares of the first compressed frame on the selected modes) against closed
forms on data built from known exponentials."""

import numpy as np

from oracle.cdmd import fit, select_background


def _planted(p=40, m=60, seed=0, orth=True):
    """Y_full = sum_q a_q phi_q lambda_q^t with known lambda: a static mode (lambda = 1),
    a slowly decaying one (lambda = e^-0.05), an oscillating pair (e^{+-i 0.7}) with
    conjugate coefficients (real data).  Columns phi orthonormal if orth."""
    rng = np.random.default_rng(seed)
    Q = np.linalg.qr(rng.standard_normal((p, 4)))[0] if orth else rng.standard_normal((p, 4))
    t = np.arange(m)
    static = 5.0 * Q[:, [0]] * np.ones((1, m))
    decay = 3.0 * Q[:, [1]] * np.exp(-0.05 * t)[None, :]
    osc = 2.0 * (Q[:, [2]] * np.cos(0.7 * t)[None, :] + Q[:, [3]] * np.sin(0.7 * t)[None, :])
    return static, decay, osc


def test_select_background_is_a_threshold_in_index_order():
    om = np.array([0.3j, -0.001, 0.02 + 0.01j, -0.3j, 0.0, 1.0])
    assert select_background(om, 0.01) == [1, 4]
    assert select_background(om, 0.1) == [1, 2, 4]
    assert select_background(om, 10.0, cap=3) == [0, 1, 2]
    assert select_background(om, 0.0) == []


def test_static_mode_only_recovers_the_static_component():
    # orthonormal planted modes: the least-squares amplitude on the static mode is the
    # static component itself, so the background of frame 1 is exactly 5 phi_0
    static, decay, osc = _planted()
    Y = static + decay + osc
    mdl = fit(Y, 4, 4, omega_eps=0.01)
    om = mdl["omega"]
    assert len(mdl["support"]) == 1
    j = mdl["support"][0]
    assert abs(om[j]) < 1e-9
    bg = (mdl["PhiY"][:, mdl["support"]] @ mdl["beta"]).real
    assert np.allclose(bg, static[:, 0], atol=1e-9)


def test_all_modes_reconstruct_the_first_frame_exactly():
    # every planted frequency below eps: the selected modes span y1, residual 0; the
    # selected omegas are the planted ones
    static, decay, osc = _planted(orth=False, seed=3)
    Y = static + decay + osc
    mdl = fit(Y, 4, 4, omega_eps=1.0)
    S = mdl["support"]
    assert len(S) == 4
    y1 = Y[:, 0]
    assert np.linalg.norm(mdl["PhiY"][:, S] @ mdl["beta"] - y1) < 1e-9 * np.linalg.norm(y1)
    got = np.sort_complex(np.round(mdl["omega"][S], 9))
    want = np.sort_complex(np.round(np.array([0.0, -0.05, 0.7j, -0.7j]), 9))
    assert np.allclose(got, want, atol=1e-8)


def test_decaying_mode_joins_above_its_rate():
    static, decay, osc = _planted(seed=5)
    Y = static + decay + osc
    assert len(fit(Y, 4, 4, omega_eps=0.04)["support"]) == 1     # |omega| = 0.05 excluded
    mdl = fit(Y, 4, 4, omega_eps=0.06)
    assert len(mdl["support"]) == 2                               # static + decay, not the pair
    bg = (mdl["PhiY"][:, mdl["support"]] @ mdl["beta"]).real
    assert np.allclose(bg, static[:, 0] + decay[:, 0], atol=1e-9)


def test_selection_is_capped_at_K():
    # reading R24: at most K background modes (||beta||_0 <= K, as for OMP); with every
    # planted frequency below eps and K = 2 the first two selected modes in mode order are
    # kept and their amplitudes are the least-squares fit of y1 on those two alone
    static, decay, osc = _planted(orth=False, seed=3)
    Y = static + decay + osc
    full = fit(Y, 4, 4, omega_eps=1.0)
    capped = fit(Y, 4, 2, omega_eps=1.0)
    assert capped["support"] == full["support"][:2]
    D = capped["PhiY"][:, capped["support"]]
    y1 = Y[:, 0]
    r = y1 - D @ capped["beta"]
    assert np.linalg.norm(D.conj().T @ r) < 1e-9 * np.linalg.norm(D) * np.linalg.norm(y1)
