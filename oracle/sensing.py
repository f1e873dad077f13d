"""Measurement matrices C in R^{p x n} and the sketch Y = C X (oracle side).

TEST INFRASTRUCTURE — see oracle/__init__.py.

Paper: C in R^{p x n} (the "rand(p,m)" of Alg. 1 step 2, is read
as p x n, reading R1).  Distributions (§3.3):
  * single pixel   C = R: p rows of I_n drawn without replacement
  * sparse         c_ij = +1 w.p. 1/(2s), 0 w.p. 1-1/s, -1 w.p. 1/(2s),
                   s = n / log(n) by default
  * Rademacher     c_ij = +-1 (Bernoulli; the s = 1 case of P:386-393)
  * Gaussian       c_ij ~ N(0,1), rounded to bf16 (north_star; reading R7)

The stream layouts that turn Philox words into these entries are fixed in
DESIGN.md §3 (they are ours, the paper fixes only the distributions):

  single pixel : row r = pi(r), pi a Philox-keyed bijection of [0, n)
                 (6-round balanced Feistel on 2h-bit words, cycle-walked;
                  round i: F_i(R) = Philox(ctr=(R, i, 0, 1))[0] mod 2^h)
  sparse       : row r walks the pixels with geometric gaps;
                 draw j: w = Philox(ctr=(j, r, 0, 2)),
                 u = (((w1 & 0x1FFFFF) << 32 | w0) + 0.5) * 2^-53,
                 g = floor(log(u) / log1p(-1/s)), pos = prev + 1 + g (first: g),
                 sign = +1 if (w2 & 1) == 0 else -1, stop when pos >= n
  Rademacher   : c_ri = +1 if bit (i mod 128) of Philox(ctr=(i // 128, r, 0, 3)) is 0
                 (bits 0-31 in w0, ... , 96-127 in w3), else -1
  Gaussian     : c_ri = T[u16], u16 = 16-bit half (i mod 8) of
                 Philox(ctr=(i // 8, r, 0, 4)) (w0 low half is slot 0, w0 high
                 half slot 1, ...), T[j] = bf16_RNE(Phi^-1((j + 1/2) / 2^16))
  SRFT         : C = R F D, realified (reading R25): p/2
                 frequencies f_r = pi'(r) (the Feistel bijection of single pixel with
                 tag 5), phases phi_i = 16-bit half (i mod 8) of Philox(ctr=(i // 8, 0,
                 0, 6)) (D = exp(2 pi i phi / 2^16), uniform on the 2^16-th roots of
                 unity); entry phase index q_ri = (phi_i - floor(2^16 ((f_r i) mod n) / n))
                 mod 2^16; row r < p/2: fp16_RNE(cos(2 pi q / 2^16)) (Re), row p/2 + r:
                 fp16_RNE(sin(2 pi q / 2^16)) (Im)

Key = (seed & 0xffffffff, seed >> 32).  Columns are indexed by the GLOBAL pixel
index, so slabs of a pixel-sharded video sum to the full sketch.

Pins (tests/test_oracle_sensing.py): Random123 KAT for Philox; permutation at
p = n; exact brute-force C X against the materialised dense C; entry
frequencies inside binomial confidence intervals; E||Cx||^2 identities;
Gaussian table symmetry / moments / closed-form quantiles.
"""

import numpy as np
from scipy.special import ndtri

from .philox import philox4x32_10, seed_key

SPIXEL, SPARSE, RADEMACHER, GAUSSIAN, SRFT = 0, 1, 2, 3, 4
KIND_NAMES = {SPIXEL: "spixel", SPARSE: "sparse", RADEMACHER: "rademacher", GAUSSIAN: "gaussian", SRFT: "srft"}
TAG = {SPIXEL: 1, SPARSE: 2, RADEMACHER: 3, GAUSSIAN: 4, SRFT: 5}
TAG_SRFT_PHASE = 6
FEISTEL_ROUNDS = 6


def default_s(n):
    """Very sparse rate s = n / log(n), natural log (reading R6)."""
    return n / np.log(n)


# ----------------------------------------------------------------- single pixel
def _feistel_halfbits(n):
    bits = max(1, int(n - 1).bit_length())
    return (bits + 1) // 2


def _feistel_encrypt(x, h, k0, k1, tag=TAG[SPIXEL]):
    mask = np.uint64((1 << h) - 1)
    L = x >> np.uint64(h)
    R = x & mask
    for i in range(FEISTEL_ROUNDS):
        f = philox4x32_10(R, i, 0, tag, k0, k1)[0] & mask
        L, R = R, L ^ f
    return (L << np.uint64(h)) | R


def _feistel_perm(n, p, seed, tag):
    k0, k1 = seed_key(seed)
    h = _feistel_halfbits(n)
    out = np.arange(p, dtype=np.uint64)
    todo = np.ones(p, dtype=bool)
    while todo.any():
        out[todo] = _feistel_encrypt(out[todo], h, k0, k1, tag)
        todo = out >= np.uint64(n)
    return out.astype(np.int64)


def spixel_rows(n, p, seed):
    """Row indices of C = R: pi(0), ..., pi(p-1), pi a bijection of [0, n).

    Sampling p pixels without replacement: distinct because pi is a
    bijection (Feistel networks are invertible; cycle walking restricts a
    bijection of [0, 2^2h) to one of [0, n)).
    """
    k0, k1 = seed_key(seed)
    h = _feistel_halfbits(n)
    x = np.arange(p, dtype=np.uint64)
    out = x.copy()
    todo = np.ones(p, dtype=bool)
    while todo.any():
        out[todo] = _feistel_encrypt(out[todo], h, k0, k1)
        todo = out >= np.uint64(n)
    return out.astype(np.int64)


# ----------------------------------------------------------------------- sparse
def sparse_rows(n, p, s, seed):
    """List over rows r of (positions int64[], signs int8[]) of the non-zeros.

    Gaps between consecutive non-zeros of an i.i.d. Bernoulli(1/s) row are
    geometric: P(g >= k) = (1 - 1/s)^k, sampled by inversion
    g = floor(log u / log(1 - 1/s)); each non-zero is +-1 with equal
    probability.
    """
    k0, k1 = seed_key(seed)
    lq = np.log1p(-1.0 / s)
    rows = []
    batch = 64
    for r in range(p):
        pos_list, sgn_list = [], []
        prev = -1
        j0 = 0
        done = False
        while not done:
            j = np.arange(j0, j0 + batch, dtype=np.uint64)
            w0, w1, w2, _ = philox4x32_10(j, r, 0, TAG[SPARSE], k0, k1)
            U = ((w1 & np.uint64(0x1FFFFF)) << np.uint64(32)) | w0
            u = (U.astype(np.float64) + 0.5) * 2.0 ** -53
            g = np.floor(np.log(u) / lq)
            for gi, sb in zip(g, w2):
                pos = prev + 1 + int(gi)
                if pos >= n:
                    done = True
                    break
                pos_list.append(pos)
                sgn_list.append(1 if (int(sb) & 1) == 0 else -1)
                prev = pos
            j0 += batch
        rows.append((np.array(pos_list, dtype=np.int64), np.array(sgn_list, dtype=np.int8)))
    return rows


# ------------------------------------------------------------------- Rademacher
def rademacher_block(rows, cols, seed):
    """Dense C[rows][:, cols] entries in {-1, +1} (int8)."""
    k0, k1 = seed_key(seed)
    rows = np.asarray(rows, dtype=np.uint64)[:, None]
    cols = np.asarray(cols, dtype=np.uint64)[None, :]
    w = philox4x32_10(cols >> np.uint64(7), rows, 0, TAG[RADEMACHER], k0, k1)
    b = cols & np.uint64(127)
    word = np.choose((b >> np.uint64(5)).astype(np.int64), w)
    bit = (word >> (b & np.uint64(31))) & np.uint64(1)
    return (1 - 2 * bit.astype(np.int64)).astype(np.int8)


# --------------------------------------------------------------------- Gaussian
def _bf16_rne(x):
    """Round fp64 values to the nearest bfloat16 (8 significant bits), ties to even."""
    m, e = np.frexp(np.asarray(x, dtype=np.float64))  # x = m * 2^e, 0.5 <= |m| < 1
    return np.ldexp(np.round(np.ldexp(m, 8)), e - 8)  # np.round: half to even


def gaussian_table():
    """T[j] = bf16_RNE(Phi^{-1}((j + 1/2) / 2^16)), j = 0 .. 65535 (fp64 values)."""
    j = np.arange(65536, dtype=np.float64)
    return _bf16_rne(ndtri((j + 0.5) / 65536.0))


_GT = None


def gaussian_block(rows, cols, seed):
    """Dense C[rows][:, cols] entries, bf16-valued N(0,1) (as fp64)."""
    global _GT
    if _GT is None:
        _GT = gaussian_table()
    k0, k1 = seed_key(seed)
    rows = np.asarray(rows, dtype=np.uint64)[:, None]
    cols = np.asarray(cols, dtype=np.uint64)[None, :]
    w = philox4x32_10(cols >> np.uint64(3), rows, 0, TAG[GAUSSIAN], k0, k1)
    slot = cols & np.uint64(7)
    word = np.choose((slot >> np.uint64(1)).astype(np.int64), w)
    u16 = (word >> (np.uint64(16) * (slot & np.uint64(1)))) & np.uint64(0xFFFF)
    return _GT[u16.astype(np.int64)]


# ------------------------------------------------------------------------- SRFT
def srft_freqs(n, nf, seed):
    """R of C = R F D: nf distinct frequencies of [0, n), drawn without
    replacement through the Feistel bijection (tag 5)."""
    return _feistel_perm(n, nf, seed, TAG[SRFT])


def srft_phases(cols, seed):
    """D: phase indices phi_i in [0, 2^16) of the unit-circle diagonal,
    d_i = exp(2 pi i phi_i / 2^16): the 16-bit half (i mod 8) of Philox(i // 8, 0, 0, 6)."""
    k0, k1 = seed_key(seed)
    cols = np.asarray(cols, dtype=np.uint64)
    w = philox4x32_10(cols >> np.uint64(3), 0, 0, TAG_SRFT_PHASE, k0, k1)
    slot = cols & np.uint64(7)
    word = np.choose((slot >> np.uint64(1)).astype(np.int64), w)
    return ((word >> (np.uint64(16) * (slot & np.uint64(1)))) & np.uint64(0xFFFF)).astype(np.int64)


def srft_table():
    """(cos, sin) of 2 pi j / 2^16, j = 0 .. 65535, as fp16 (RNE) values in fp64, built
    from the quarter wave Q[r] = fp16(cos(2 pi r / 2^16)), r = 0 .. 2^14, by the exact
    symmetries cos(pi/2 qd + t) = (Q[r], -Q[2^14 - r], -Q[r], Q[2^14 - r]) for quadrant
    qd = 0..3 (t = 2 pi r / 2^16), and sin(x) = cos(x - pi/2)."""
    r = np.arange(16385, dtype=np.float64)
    Q = np.cos(2.0 * np.pi * r / 65536.0).astype(np.float16).astype(np.float64)
    j = np.arange(65536)
    qd, rr = j >> 14, j & 16383
    idx = np.where(qd & 1, 16384 - rr, rr)
    cos = np.where((qd == 1) | (qd == 2), -Q[idx], Q[idx])
    return cos, cos[(j - 16384) % 65536]


_ST = None


def srft_block(rows, cols, seed, n, p):
    """Dense rows of the realified SRFT (reading R25): C[r] = Re(R F D)[r] for r < p/2,
    Im(R F D)[r - p/2] for r >= p/2, with F(f, i) = exp(-2 pi i f i / n) (the
    "/m" of the garbled formula read as /n) and the phase quantised to 2^-16 turn."""
    global _ST
    if _ST is None:
        _ST = srft_table()
    if p % 2:
        raise ValueError("SRFT needs an even p (p/2 complex measurements)")
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    f = srft_freqs(n, p // 2, seed)[rows % (p // 2)][:, None]           # frequency of each row
    a = (f * cols[None, :]) % n                                         # (f i) mod n, < 2^23
    b = (a * 65536) // n                                                # floor(2^16 a / n)
    q = (srft_phases(cols, seed)[None, :] - b) % 65536
    re = (rows < p // 2)[:, None]
    return np.where(re, _ST[0][q], _ST[1][q])


# ------------------------------------------------------------------ dense C
def dense_C(kind, n, p, seed, s=None, rows=None):
    """Materialise C (or the given rows of it) — only for tiny n (brute-force pins)."""
    rows = np.arange(p) if rows is None else np.asarray(rows)
    if kind == SPIXEL:
        idx = spixel_rows(n, p, seed)
        C = np.zeros((len(rows), n), dtype=np.int64)
        C[np.arange(len(rows)), idx[rows]] = 1
        return C
    if kind == SPARSE:
        s = default_s(n) if s is None else s
        lists = sparse_rows(n, p, s, seed)
        C = np.zeros((len(rows), n), dtype=np.int64)
        for a, r in enumerate(rows):
            pos, sg = lists[r]
            C[a, pos] = sg
        return C
    if kind == RADEMACHER:
        return rademacher_block(rows, np.arange(n), seed).astype(np.int64)
    if kind == GAUSSIAN:
        return gaussian_block(rows, np.arange(n), seed)
    if kind == SRFT:
        return srft_block(rows, np.arange(n), seed, n, p)
    raise ValueError(kind)


# ----------------------------------------------------------------------- sketch
def sketch(X, kind, p, seed, s=None, n_total=None, pix0=0, rows=None, chunk=1 << 16):
    """Y_full = C D  (p x m), Alg. 1 step 3 / Eq..

    X : uint8 array (m, n_local), frame-major (X[t, j] = pixel pix0 + j of frame t).
    Returns int64 (integer kinds, exact) or float64 (Gaussian) array (len(rows), m).
    Columns of C are indexed by the global pixel pix0 + j.
    """
    X = np.asarray(X)
    m, n_local = X.shape
    n = n_local if n_total is None else n_total
    rows = np.arange(p) if rows is None else np.asarray(rows)
    if kind == SPIXEL:
        idx = spixel_rows(n, p, seed)[rows]
        Y = np.zeros((len(rows), m), dtype=np.int64)
        inside = (idx >= pix0) & (idx < pix0 + n_local)
        Y[inside] = X[:, idx[inside] - pix0].T.astype(np.int64)
        return Y
    if kind == SPARSE:
        s = default_s(n) if s is None else s
        lists = sparse_rows(n, p, s, seed)
        Y = np.zeros((len(rows), m), dtype=np.int64)
        for a, r in enumerate(rows):
            pos, sg = lists[r]
            sel = (pos >= pix0) & (pos < pix0 + n_local)
            Y[a] = (X[:, pos[sel] - pix0].astype(np.int64) * sg[sel].astype(np.int64)).sum(axis=1)
        return Y
    if kind in (RADEMACHER, GAUSSIAN, SRFT):
        if kind == SRFT:
            def block(r, c, sd):
                return srft_block(r, c, sd, n, p)
        else:
            block = rademacher_block if kind == RADEMACHER else gaussian_block
        acc_t = np.int64 if kind == RADEMACHER else np.float64
        Y = np.zeros((len(rows), m), dtype=acc_t)
        for c0 in range(0, n_local, chunk):
            c1 = min(n_local, c0 + chunk)
            Cb = block(rows, np.arange(pix0 + c0, pix0 + c1), seed).astype(acc_t)
            Y += Cb @ X[:, c0:c1].T.astype(acc_t)
        return Y
    raise ValueError(kind)
