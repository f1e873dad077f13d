"""Helpers shared by the GPU parity tests: tolerances from BASELINE.json's
north_star and the comparison rules of DESIGN.md §8."""

import numpy as np

# north_star: "bit-exact for the integer sketches ...; relative error <= 1e-4 for
# fp32 Y, Phi and eigenvalues; >= 99.9% pixel agreement of foreground masks, with
# disagreements allowed only within 1e-3 of the threshold."
RTOL_EIG = 1e-4
RTOL_PHI = 1e-4
RTOL_Y_GAUSS = 1e-4
MASK_AGREE = 0.999
MASK_BAND = 1e-3


def match_eigs(lam_gpu, lam_ref):
    """Greedy nearest matching; returns (perm: gpu index -> ref index, max rel error)."""
    ref = list(range(len(lam_ref)))
    perm = [-1] * len(lam_gpu)
    worst = 0.0
    order = np.argsort(-np.abs(lam_gpu))
    for i in order:
        d = [abs(lam_gpu[i] - lam_ref[j]) for j in ref]
        a = int(np.argmin(d))
        j = ref.pop(a)
        perm[i] = j
        worst = max(worst, d[a] / max(abs(lam_ref[j]), 1e-300))
    return perm, worst


def unfold(F, pair):
    """Folded real columns (ncols x n) -> complex (n x ncols)."""
    F = np.asarray(F, dtype=np.float64)
    k = len(pair)
    out = np.empty((F.shape[1], k), dtype=np.complex128)
    for c in range(k):
        if pair[c] == 0:
            out[:, c] = F[c]
        elif pair[c] == 1:
            out[:, c] = F[c] + 1j * F[c + 1]
        else:
            out[:, c] = F[c - 1] - 1j * F[c]
    return out


def phase_aligned_rel(a, b):
    """min over unit phases u of ||a - u b|| / ||b||."""
    ip = np.vdot(b, a)
    u = ip / abs(ip) if abs(ip) > 0 else 1.0
    return np.linalg.norm(a - u * b) / max(np.linalg.norm(b), 1e-300)


def well_separated(lam, i, tol=1e-8):
    return all(abs(lam[i] - lam[j]) > tol * max(1.0, abs(lam[i])) for j in range(len(lam)) if j != i)


def supports_equal_mod_conj(sup_gpu, pair_gpu, perm, sup_ref, pair_ref):
    """Supports compared as sets of eigen-units (a mode and its conjugate partner
    are one unit), GPU indices mapped to oracle indices by eigenvalue matching."""
    def unit(i, pair):
        return i - 1 if pair[i] < 0 else i
    g = sorted(unit(perm[i], pair_ref) for i in sup_gpu)
    o = sorted(unit(i, pair_ref) for i in sup_ref)
    return g == o


def mask_agreement(mask_gpu, mask_ref, resid_ref, tau):
    """Fraction of agreeing pixels and whether every disagreement lies within
    MASK_BAND of the threshold (|resid_ref - tau| <= MASK_BAND)."""
    dis = mask_gpu != mask_ref
    frac = 1.0 - dis.mean()
    ok_band = bool(np.all(np.abs(resid_ref[dis] - tau) <= MASK_BAND))
    return frac, ok_band, int(dis.sum())
