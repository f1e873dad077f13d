"""Compressed DMD, Algorithm 1 of arXiv 1512.04205, step by step (oracle side).

TEST INFRASTRUCTURE — see oracle/__init__.py.  fp64 / complex128 throughout;
numpy.linalg (LAPACK) is used only for the small SVD / eig / lstsq steps.

Steps, in the paper's order and notation:
  fit()        Alg. 1 steps 1, 4, 6, 7 + Remark 3 OMP
               + omega = log(lambda)/dt; the target rank fixed, or
               (rank="gd") chosen by the Gavish-Donoho optimal hard threshold
               (Remark 2; evaluation settings P:573) via optimal_rank()
  modes()      Alg. 1 step 8, Eq. cDMDModes  Phi = X' V S^-1 W
  amplitudes() Alg. 1 step 9, b = lstsq(Phi, x_1) on the full-state modes,
               pinned in tests/test_oracle_amplitudes.py
  background() Eq. DMDTerms: L = Re sum_{p in S} b_p phi_p lambda_p^{t-1}
               (dynamic) or x_BG = Re Phi beta (static)
  mask()       Eq. thres: 1 iff |x_jt - xhat_j| > tau
  median3()    the 3x3 median post-filter of the mask (Fig. 7)

Readings of silent / garbled passages are listed in DESIGN.md §4 (R1..R20) and
cited inline as "reading Rn".

Pins (tests/test_oracle_dmd.py, tests/test_oracle_omp.py): C = I reproduces
exact DMD (pinv formulation); uint8-exact periodic videos give lambda = 1, +-i
exactly; planted exponentials; static video; x_t = 2^(t-1)[1,1] -> lambda = 2;
Phi_Y = C Phi (linearity); OMP = exhaustive search for K = 1 and planted
supports; OMP residual orthogonality; mask monotone in tau and hand cases.
"""

import numpy as np

RANK_RTOL = 1e-6      # reading R10: drop sigma_j <= RANK_RTOL * sigma_1
OMP_STOP_RTOL = 1e-6  # reading R12: stop OMP early if ||r|| <= OMP_STOP_RTOL ||y1||
TIE_RTOL = 1e-9       # reading R13: OMP scores within TIE_RTOL of the max tie -> lowest index


def canonical_eig(A):
    """eig(A) (Alg. 1 step 7) in canonical order and normalisation.

    Order (reading R11): units sorted by |lambda| descending; a real eigenvalue
    is one unit, a conjugate pair is one unit listed as (Im > 0, Im < 0).
    Normalisation: unit 2-norm, largest-magnitude component real positive; the
    Im < 0 member of a pair is the exact conjugate of its partner.
    Returns lam (k,), W (k, k) complex, pair (k,) int: +1 first of pair,
    -1 second of pair, 0 real.
    """
    lam, W = np.linalg.eig(A)
    k = len(lam)
    used = np.zeros(k, dtype=bool)
    units = []
    for i in range(k):
        if used[i]:
            continue
        used[i] = True
        if lam[i].imag == 0.0:
            units.append((abs(lam[i]), 0, i, None))
            continue
        # LAPACK returns conjugate pairs as exact conjugates; find the partner.
        cand = [j for j in range(k) if not used[j] and lam[j] == np.conj(lam[i])]
        j = cand[0]
        used[j] = True
        a, b = (i, j) if lam[i].imag > 0 else (j, i)
        units.append((abs(lam[a]), 1, a, b))
    units.sort(key=lambda u: (-u[0], u[1]))
    order, pair = [], []
    for _, isp, a, b in units:
        if isp:
            order += [a, b]
            pair += [1, -1]
        else:
            order.append(a)
            pair.append(0)
    lam = lam[order].astype(np.complex128)
    W = W[:, order].astype(np.complex128)
    pair = np.array(pair, dtype=np.int64)
    for j in range(k):
        if pair[j] == -1:
            lam[j] = np.conj(lam[j - 1])
            W[:, j] = np.conj(W[:, j - 1])
            continue
        if pair[j] == 0:
            lam[j] = complex(lam[j].real, 0.0)
            W[:, j] = W[:, j].real
        w = W[:, j] / np.linalg.norm(W[:, j])
        i = int(np.argmax(np.abs(w)))
        W[:, j] = w * (np.conj(w[i]) / abs(w[i]))
    return lam, W, pair


def omp(D, y, K, stop_rtol=OMP_STOP_RTOL, tie_rtol=TIE_RTOL):
    """Orthogonal matching pursuit (Remark 3).

    Greedy: select the column with the highest normalised correlation
    |d_j^H r| / ||d_j|| with the current residual; project y orthogonally on
    the span of the selected columns (least squares); recompute the residual;
    repeat until K non-zeros (reading R12: ||beta||_0 <= K, the paper's
    "K = 10 non-zero entries").
    Returns (support list, beta complex array aligned with support).
    """
    D = np.asarray(D, dtype=np.complex128)
    y = np.asarray(y, dtype=np.complex128)
    norms = np.linalg.norm(D, axis=0)
    ynorm = np.linalg.norm(y)
    r = y.copy()
    S = []
    beta = np.zeros(0, dtype=np.complex128)
    for _ in range(min(K, D.shape[1])):
        if ynorm == 0.0 or np.linalg.norm(r) <= stop_rtol * ynorm:
            break
        score = np.full(D.shape[1], -np.inf)
        ok = norms > 0
        score[ok] = np.abs(D[:, ok].conj().T @ r) / norms[ok]
        score[S] = -np.inf
        best = score.max()
        if not np.isfinite(best) or best <= 0.0:
            break
        j = int(np.flatnonzero(score >= best * (1.0 - tie_rtol))[0])
        S.append(j)
        beta = np.linalg.lstsq(D[:, S], y, rcond=None)[0]
        r = y - D[:, S] @ beta
    return S, beta


def omega_beta(beta):
    """Gavish-Donoho unknown-noise coefficient omega(beta) ~ 0.56 b^3 - 0.95 b^2 + 1.82 b + 1.43
    (the cubic approximation of the cited work; SPEC optimal_rank)."""
    return 0.56 * beta ** 3 - 0.95 * beta ** 2 + 1.82 * beta + 1.43


def optimal_rank(s, rows, cols):
    """Remark 2: number of singular values above tau = omega(beta) median(s),
    beta = min(rows, cols) / max(rows, cols); s = ALL singular values of the rows x cols
    matrix.  At least 1."""
    s = np.asarray(s, dtype=np.float64)
    if s.size == 0:
        raise ValueError("empty singular-value vector")
    beta = min(rows, cols) / max(rows, cols)
    tau = omega_beta(beta) * np.median(s)
    return max(int(np.count_nonzero(s > tau)), 1)


def select_background(omega, eps, cap=32):
    """Background modes by frequency (modes with |omega_p| ~ 0 model the
    slowly varying background): the columns j with |omega_j| < eps, in index order,
    at most `cap` (fit passes K: the model holds at most K background modes, reading R24)."""
    return [j for j in range(len(omega)) if abs(omega[j]) < eps][:cap]


def fit(Yfull, k, K, dt=1.0, rank_rtol=RANK_RTOL, rank="fixed", omega_eps=None):
    """cDMD small solve from the full sketch Y_full = C D (p x m).

    Y = Y_full[:, :m-1], Y' = Y_full[:, 1:] (Eq. FullData; reading R2).
    Alg. 1: step 4 truncated SVD (Eq. svd); step 6
    A~ = U* Y' V S^-1; step 7 eig;
    Phi_Y = Y' V S^-1 W; Remark 3: beta = omp(Phi_Y, y1);
    omega = log(lambda)/dt (principal branch, reading R15).
    omega_eps: select the background by |omega| < omega_eps (select_background)
    instead of OMP, beta = least squares of y1 on those compressed modes.
    """
    Yfull = np.asarray(Yfull, dtype=np.float64)
    p, m = Yfull.shape
    Y, Yp = Yfull[:, :m - 1], Yfull[:, 1:]
    U, s, Vh = np.linalg.svd(Y, full_matrices=False)
    k = min(k, len(s))
    if rank == "gd":      # Remark 2: k = optimal hard-threshold rank, at most k
        k = min(k, optimal_rank(s, p, m - 1))
    elif rank != "fixed":
        raise ValueError(rank)
    U, s, V = U[:, :k], s[:k], Vh[:k].T
    keep = s > rank_rtol * s[0] if s.size and s[0] > 0 else np.zeros(k, dtype=bool)
    k_eff = int(np.count_nonzero(keep))
    if k_eff == 0:
        raise FloatingPointError("every singular value dropped")
    U, s, V = U[:, :k_eff], s[:k_eff], V[:, :k_eff]
    Atilde = U.T @ Yp @ V @ np.diag(1.0 / s)
    lam, W, pair = canonical_eig(Atilde)
    M = V @ np.diag(1.0 / s) @ W                       # V S^-1 W, (m-1) x k
    PhiY = Yp @ M                                      # compressed modes, p x k
    y1 = Y[:, 0]                                       # first compressed frame
    omega = np.log(lam) / dt
    if omega_eps is None:
        support, beta = omp(PhiY, y1, K)
    else:
        support = select_background(omega, omega_eps, cap=K)   # ||beta||_0 <= K (reading R24)
        beta = (np.linalg.lstsq(PhiY[:, support].astype(np.complex128), y1.astype(np.complex128), rcond=None)[0]
                if support else np.zeros(0, dtype=np.complex128))
    return dict(k=k, k_eff=k_eff, sigma=s, V=V, U=U, Atilde=Atilde, lam=lam, W=W,
                pair=pair, M=M, PhiY=PhiY, support=list(support), beta=beta,
                omega=omega, dt=dt, m=m, p=p)


def fold(M, pair):
    """Real 'conjugate-folded' columns of a complex matrix whose columns come in
    conjugate pairs: real mode -> Re; pair (j, j+1) -> Re, Im of j."""
    F = np.empty(M.shape, dtype=np.float64)
    for j in range(M.shape[1]):
        F[:, j] = M[:, j].real if pair[j] >= 0 else M[:, j - 1].imag
    return F


def modes(X, M):
    """Phi = X' V S^-1 W = X' M (Eq. cDMDModes), complex128.

    X : uint8 (m, n) frame-major; X' = frames 2..m.
    """
    Xp = np.asarray(X[1:], dtype=np.float64)           # (m-1, n)
    return Xp.T @ M                                    # (n, k)


def amplitudes(X, Phi):
    """b = lstsq(Phi, x_1) (Alg. 1 step 9: "Compute amplitudes using x_1 as
    initial condition"), complex128 (k,).  X uint8 (m, n) frame-major, x_1 = frame 1
    (P:71); Phi (n, k) complex as returned by modes()."""
    x1 = np.asarray(X[0], dtype=np.float64).astype(np.complex128)
    return np.linalg.lstsq(np.asarray(Phi, dtype=np.complex128), x1, rcond=None)[0]


def background_static(Phi, model):
    """x_BG = Re(Phi beta) (real part per footnote P:193)."""
    S = model["support"]
    return (Phi[:, S] @ model["beta"]).real


def background_dynamic(Phi, model, t0=0, nt=None):
    """L[:, t] = Re sum_{p in S} beta_p phi_p lambda_p^(t-1), t = t0+1 .. t0+nt
    (Eq. DMDTerms P:185-193 with Eq. omegaj; lambda^(t-1) = exp((t-1) Log lambda))."""
    S = model["support"]
    nt = model["m"] - t0 if nt is None else nt
    t = np.arange(t0, t0 + nt, dtype=np.float64)         # t - 1
    lamS = model["lam"][S]
    vander = np.exp(np.outer(np.log(lamS), t))         # K x nt
    return (Phi[:, S] @ (model["beta"][:, None] * vander)).real   # n x nt


def mask(X, L, tau):
    """Foreground mask (Eq. thres): 1 iff |x_jt - L_jt| > tau (strict;
    reading R16/R17).  X uint8 (m, n); L (n,) static or (n, m) dynamic.
    Returns bool (m, n)."""
    Xf = np.asarray(X, dtype=np.float64)
    L = np.asarray(L, dtype=np.float64)
    Lt = L[None, :] if L.ndim == 1 else L.T
    return np.abs(Xf - Lt) > tau


def median3(Mb, width, height):
    """3x3 spatial median of each frame's binary mask (the "in addition median filtered
    foreground mask" of Fig. 7; SPEC median3).  On a binary image the median of
    the 9 values is the majority: bit = 1 iff at least 5 of the 3x3 neighbourhood are
    set.  Outside the image counts as 0 (zero padding, reading R22).
    Mb: bool (m, n) with n = width * height, pixel j = y * width + x.  Returns bool (m, n)."""
    Mb = np.asarray(Mb, dtype=bool)
    m, n = Mb.shape
    if n != width * height:
        raise ValueError("mask is not whole frames")
    F = Mb.reshape(m, height, width).astype(np.int32)
    P = np.zeros((m, height + 2, width + 2), dtype=np.int32)
    P[:, 1:-1, 1:-1] = F
    cnt = np.zeros_like(F)
    for dy in range(3):
        for dx in range(3):
            cnt += P[:, dy:dy + height, dx:dx + width]
    return (cnt >= 5).reshape(m, n)


def pack_mask(Mb):
    """Bit-pack a bool (m, n) mask: bit j%32 of uint32 word (t, j//32)."""
    m, n = Mb.shape
    nw = (n + 31) // 32
    pad = np.zeros((m, nw * 32), dtype=bool)
    pad[:, :n] = Mb
    by = np.packbits(pad.reshape(m, nw, 4, 8), axis=-1, bitorder="little")[..., 0]
    return by.view("<u4").reshape(m, nw) if by.flags.c_contiguous else np.ascontiguousarray(by).view("<u4").reshape(m, nw)


def unpack_mask(W, n):
    """Inverse of pack_mask: uint32 (m, nw) -> bool (m, n)."""
    W = np.ascontiguousarray(np.asarray(W, dtype="<u4"))
    m = W.shape[0]
    by = W.view(np.uint8).reshape(m, -1)
    return np.unpackbits(by, axis=1, bitorder="little")[:, :n].astype(bool)


def cdmd(X, kind, p, k, K, seed=0, s=None, tau=25.0, dynamic=True, dt=1.0):
    """Whole pipeline on a small video: sketch -> fit -> modes -> background -> mask."""
    from .sensing import sketch
    Yfull = sketch(X, kind, p, seed, s=s)
    model = fit(Yfull, k, K, dt=dt)
    Phi = modes(X, model["M"])
    L = background_dynamic(Phi, model) if dynamic else background_static(Phi, model)
    return dict(Y=Yfull, model=model, Phi=Phi, L=L, mask=mask(X, L, tau))
