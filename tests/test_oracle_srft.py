"""Pins for the oracle's SRFT sensing matrix C = R F D, realified
(reading R25): each of the p/2 complex measurements gives the rows Re and Im.

Checked against an independent complex construction of R F D written out from the
paper's definition (R: rows of the identity without replacement; F(j, k) =
exp(-2 pi i j k / n); D: unit-circle diagonal), within the stated quantisation (phase
to 2^-16 turn, entries to fp16), plus the structural facts the paper relies on."""

import math

import numpy as np
import pytest

from oracle import cdmd as OD
from oracle import sensing as S
from oracle.philox import philox4x32_10, seed_key


def _exact_rfd(n, nf, seed):
    """R F D in complex128 from the definitions: R picks rows f_r, F is the unnormalised
    DFT, D = diag(exp(2 pi i phi_k / 2^16)) with the same random phases."""
    f = S.srft_freqs(n, nf, seed)
    k = np.arange(n)
    k0, k1 = seed_key(seed)
    phi = np.empty(n, dtype=np.int64)
    for i in range(n):   # phases straight from Philox, one entry at a time
        w = philox4x32_10(np.uint64(i // 8), 0, 0, 6, k0, k1)
        word = int(w[(i % 8) // 2])
        phi[i] = (word >> (16 * (i % 2))) & 0xFFFF
    F = np.exp(-2j * np.pi * np.outer(f, k) / n)
    return F * np.exp(2j * np.pi * phi / 65536.0)[None, :]


@pytest.mark.parametrize("n,p,seed", [(37, 10, 3), (128, 64, 0), (1000, 40, 7)])
def test_entries_match_the_complex_definition(n, p, seed):
    C = S.dense_C(S.SRFT, n, p, seed)
    E = _exact_rfd(n, p // 2, seed)
    # phase quantised to 2^-16 turn (|e^{ia} - e^{ib}| <= |a - b|) plus fp16 rounding
    tol = 2 * np.pi / 65536 + 2.0 ** -11
    assert np.max(np.abs(C[:p // 2] - E.real)) <= tol
    assert np.max(np.abs(C[p // 2:] - E.imag)) <= tol


def test_frequencies_without_replacement():
    for n in (1, 5, 97, 1024):
        f = S.srft_freqs(n, n, 11)
        assert sorted(f.tolist()) == list(range(n))


def test_table_values():
    c, s = S.srft_table()
    assert c[0] == 1.0 and s[0] == 0.0 and c[32768] == -1.0 and s[16384] == 1.0
    j = np.arange(1, 65536)
    assert np.array_equal(c[j], c[65536 - j]) and np.array_equal(s[j], -s[65536 - j])   # parity of cos / sin
    for jj in (1, 777, 12345, 40000, 65535):   # independent evaluation, fp16 rounding by struct
        ang = 2 * math.pi * jj / 65536
        assert c[jj] == float(np.float16(math.cos(ang))) and s[jj] == float(np.float16(math.sin(ang)))


def test_all_frequencies_give_nearly_orthogonal_columns():
    # p/2 = n: R = I, so (RFD)^H (RFD) = n I exactly; realified, Re(C^H C) = C_re^T C_re +
    # C_im^T C_im = n I, up to the quantisation of the entries
    n = 64
    C = S.dense_C(S.SRFT, n, 2 * n, 5)
    G = C.T @ C / n
    assert np.max(np.abs(G - np.eye(n))) <= 4 * (2 * np.pi / 65536 + 2.0 ** -11)


def test_sketch_equals_dense_product_and_slabs_add_up():
    from synth.scene import make_video
    X = make_video(40, 30, 9, seed=2, noise=2.0, n_rects=1)
    n = X.shape[1]
    p = 24
    C = S.dense_C(S.SRFT, n, p, 4)
    Y = S.sketch(X, S.SRFT, p, 4)
    assert np.allclose(Y, C @ X.T.astype(np.float64), rtol=0, atol=1e-9 * np.abs(Y).max())
    Ys = S.sketch(X[:, :500], S.SRFT, p, 4, n_total=n) + S.sketch(X[:, 500:], S.SRFT, p, 4, n_total=n, pix0=500)
    assert np.allclose(Ys, Y, rtol=0, atol=1e-9 * np.abs(Y).max())


def test_srft_cdmd_recovers_the_periodic_eigenvalues():
    """A full-rank realified SRFT keeps the column space of the data, so cDMD on the
    uint8 4-periodic video gives lambda = {1, i, -i} (here to the quantisation level)."""
    from synth.scene import make_video
    X = make_video(24, 16, 30, seed=1, noise=0.0, n_rects=0)
    Y = S.sketch(X, S.SRFT, 40, 9)
    mdl = OD.fit(Y, 3, 1)
    lam = np.sort_complex(mdl["lam"])
    assert np.allclose(lam, np.sort_complex(np.array([1.0, 1j, -1j])), atol=1e-9)
