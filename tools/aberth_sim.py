"""Aberth-Ehrlich eigenvalue study for the small nonsymmetric eig of the fit (host-side
NumPy, not on the product path).

All k eigenvalues of the upper Hessenberg form H of A-tilde are iterated at once
(Aberth-Ehrlich: z_i <- z_i - N_i / (1 - N_i sum_{j != i} 1/(z_i - z_j)), N_i = p/p'),
with p'/p evaluated by Hyman's method (the backward recurrence through the subdiagonal,
x_n = 1, x_{i-1} = -(sum_{j >= i} (H - zI)_{ij} x_j) / h_{i,i-1}, p ~ row 1's residual) and
its derivative.  Prints, per case, the iterations to convergence and the worst eigenvalue
error against numpy.linalg.eigvals.
usage: python tools/aberth_sim.py [c2_320x240_spixel c4_1080p_sparse rand50 ...]
"""
import sys

import numpy as np
import scipy.linalg

sys.path.insert(0, ".")
sys.path.insert(0, "tools")


def hyman_ratio(H, z):
    """p'(z)/p(z) of det(H - zI) for unreduced upper Hessenberg H (complex z)."""
    n = H.shape[0]
    x = np.zeros(n, complex)
    dx = np.zeros(n, complex)
    x[n - 1] = 1.0
    dx[n - 1] = 0.0
    for i in range(n - 1, 0, -1):
        row = H[i, i:].astype(complex)
        row[0] -= z
        s = row @ x[i:]
        ds = row @ dx[i:] - x[i]
        x[i - 1] = -s / H[i, i - 1]
        dx[i - 1] = -ds / H[i, i - 1]
        m = max(abs(x[i - 1]), abs(dx[i - 1]))
        if m > 1e100:
            x /= m
            dx /= m
    row = H[0, :].astype(complex)
    row[0] -= z
    f = row @ x
    df = row @ dx - x[0]
    return df / f, f


def aberth(H, iters=100, tol=1e-14, init=None):
    n = H.shape[0]
    if init is None:
        # radius: the Gershgorin-like bound of H (every eigenvalue lies within ||H||_inf)
        rad = 0.8 * np.max(np.sum(np.abs(H), axis=1))
        z = rad * np.exp(1j * (2 * np.pi * (np.arange(n) + 0.25) / n))
    else:
        z = init.copy()
    done = np.zeros(n, bool)
    for it in range(iters):
        znew = z.copy()
        for i in range(n):
            if done[i]:
                continue
            r, f = hyman_ratio(H, z[i])
            N = 1.0 / r if r != 0 else 0.0
            S = np.sum(1.0 / (z[i] - np.delete(z, i)))
            w = N / (1.0 - N * S)
            znew[i] = z[i] - w
            if abs(w) <= tol * max(abs(znew[i]), 1e-300):
                done[i] = True
        z = znew
        if done.all():
            return z, it + 1
    return z, -1


def worst_err(z, A):
    ref = np.linalg.eigvals(A)
    used = np.zeros(len(ref), bool)
    w = 0.0
    for v in z:
        d = np.abs(ref - v)
        d[used] = np.inf
        j = int(np.argmin(d))
        used[j] = True
        w = max(w, d[j] / max(abs(ref[j]), 1e-300))
    return w


def main():
    from hqr_sim import atilde
    names = sys.argv[1:] or ["c1_32x24_sparse", "c2_320x240_spixel", "rand50"]
    for nm in names:
        if nm.startswith("rand"):
            k = int(nm[4:] or 50)
            rng = np.random.default_rng(k)
            As = [(f"{nm}#{t}", rng.standard_normal((k, k)) / np.sqrt(k)) for t in range(3)]
        else:
            As = [(nm, atilde(nm))]
        for lab, A in As:
            H = scipy.linalg.hessenberg(A)
            z, it = aberth(H)
            print(f"{lab:22s} k={A.shape[0]:3d} iterations {it:4d}  worst rel err {worst_err(z, A):.2e}  "
                  f"min |h_i,i-1| {np.min(np.abs(np.diag(H, -1))):.2e}")


if __name__ == "__main__":
    main()
