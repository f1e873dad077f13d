"""Francis QR step-count study for eig.cu's hqr (host-side NumPy, not on the product path).

Runs the EISPACK hqr iteration (values only) on the Hessenberg form of a config's
A-tilde (the oracle's fit of the oracle's sketch) and of random matrices, either with
one double-shift bulge per sweep (what hqrv_kernel does) or with TWO bulges per sweep:
bulge 1 with the Francis shifts of the trailing 2 x 2 block, bulge 2 (introduced three
rows behind bulge 1 in the same sweep) with those of the 2 x 2 block above it, both
chosen before the sweep.  The pipelined order is checked against the sequential one
(sweep 1, then sweep 2) and the eigenvalues against numpy.linalg.eigvals.
Prints per case: sweeps, bulge-chase iterations (a two-bulge iteration = one slot) and
the worst eigenvalue error.
usage: python tools/hqr_sim.py [c2 c4 ...]
"""
import sys

import numpy as np
import scipy.linalg

sys.path.insert(0, ".")

EPS = 2.0 ** -52


def refl(p, q, r):
    """Householder of (p, q, r) as hqr forms it: returns (x, y, z, q', r', s)."""
    s = np.sqrt(p * p + q * q + r * r)
    if p < 0:
        s = -s
    pp = p + s
    return pp / s, q / s, r / s, q / pp, r / pp, s


def row_apply(H, k, lo_col, hi_col, c, notlast):
    x, y, z, q, r = c
    for j in range(lo_col, hi_col + 1):
        pp = H[k, j] + q * H[k + 1, j] + (r * H[k + 2, j] if notlast else 0.0)
        H[k, j] -= pp * x
        H[k + 1, j] -= pp * y
        if notlast:
            H[k + 2, j] -= pp * z


def col_apply(H, k, lo_row, hi_row, c, notlast):
    x, y, z, q, r = c
    for i in range(lo_row, hi_row + 1):
        pp = x * H[i, k] + y * H[i, k + 1] + (z * H[i, k + 2] if notlast else 0.0)
        H[i, k] -= pp
        H[i, k + 1] -= pp * q
        if notlast:
            H[i, k + 2] -= pp * r


def intro(H, m, x, y, w):
    """First column of (H - s1)(H - s2) e_m for the shifts of [[y, .], [., x]] (hqr's form)."""
    zz = H[m, m]
    r_, s_ = x - zz, y - zz
    p = (r_ * s_ - w) / H[m + 1, m] + H[m, m + 1]
    q = H[m + 1, m + 1] - zz - r_ - s_
    r = H[m + 2, m + 1]
    sc = abs(p) + abs(q) + abs(r)
    return p / sc, q / sc, r / sc


def step(H, kk, m, n, l, pqr):
    """One bulge step at kk (hqr's loop body); returns the coefficients (None: skipped)."""
    notlast = kk != n - 1
    if kk != m:
        p, q, r = H[kk, kk - 1], H[kk + 1, kk - 1], (H[kk + 2, kk - 1] if notlast else 0.0)
        xs = abs(p) + abs(q) + abs(r)
        if xs == 0.0:
            return None
        p, q, r = p / xs, q / xs, r / xs
    else:
        p, q, r = pqr
        xs = 1.0
    x, y, z, qq, rr, s = refl(p, q, r)
    if kk != m:
        H[kk, kk - 1] = -s * xs
        H[kk + 1, kk - 1] = 0.0
        if notlast:
            H[kk + 2, kk - 1] = 0.0
    elif l != m:
        H[kk, kk - 1] = -H[kk, kk - 1]
    c = (x, y, z, qq, rr)
    row_apply(H, kk, kk, n, c, notlast)
    col_apply(H, kk, l, min(n, kk + 3), c, notlast)
    return c


def sweep(H, l, n, m, pqr):
    for i in range(m + 2, n + 1):
        H[i, i - 2] = 0.0
        if i != m + 2:
            H[i, i - 3] = 0.0
    for kk in range(m, n):
        step(H, kk, m, n, l, pqr)
    return n - m


def two_sweeps_pipelined(H, l, n, pqr1, sh2):
    """Bulge 2 three rows behind bulge 1; returns the number of iteration slots."""
    for i in range(l + 2, n + 1):
        H[i, i - 2] = 0.0
        if i != l + 2:
            H[i, i - 3] = 0.0
    slots = 0
    k1 = l
    k2 = l - 3
    while k1 <= n - 1 or k2 <= n - 1:
        c1 = c2 = None
        # reflectors (bulge 1's input is read before bulge 2's column transform of this slot)
        if k1 <= n - 1:
            notlast1 = k1 != n - 1
            if k1 != l:
                p, q, r = H[k1, k1 - 1], H[k1 + 1, k1 - 1], (H[k1 + 2, k1 - 1] if notlast1 else 0.0)
                xs = abs(p) + abs(q) + abs(r)
            else:
                p, q, r = pqr1
                xs = 1.0
            if xs != 0.0:
                c1 = refl(p / xs, q / xs, r / xs) + (xs,)
        if l <= k2 <= n - 1:
            notlast2 = k2 != n - 1
            if k2 != l:
                p, q, r = H[k2, k2 - 1], H[k2 + 1, k2 - 1], (H[k2 + 2, k2 - 1] if notlast2 else 0.0)
                xs = abs(p) + abs(q) + abs(r)
            else:
                p, q, r = intro(H, l, *sh2)
                xs = 1.0
            if xs != 0.0:
                c2 = refl(p / xs, q / xs, r / xs) + (xs,)
        # left (row) transforms, then right (column) transforms
        if c1 is not None:
            x, y, z, qq, rr, s, xs = c1
            if k1 != l:
                H[k1, k1 - 1] = -s * xs
                H[k1 + 1, k1 - 1] = 0.0
                if notlast1:
                    H[k1 + 2, k1 - 1] = 0.0
            row_apply(H, k1, k1, n, (x, y, z, qq, rr), notlast1)
        if c2 is not None:
            x, y, z, qq, rr, s, xs = c2
            if k2 != l:
                H[k2, k2 - 1] = -s * xs
                H[k2 + 1, k2 - 1] = 0.0
                if notlast2:
                    H[k2 + 2, k2 - 1] = 0.0
            row_apply(H, k2, k2, n, (x, y, z, qq, rr), notlast2)
        if c1 is not None:
            col_apply(H, k1, l, min(n, k1 + 3), c1[:5], notlast1)
        if c2 is not None:
            col_apply(H, k2, l, min(n, k2 + 3), c2[:5], notlast2)
        k1 += 1
        k2 += 1
        slots += 1
    return slots


def hqr(H0, two=False, check_order=False):
    H = H0.copy()
    nn = H.shape[0]
    n = nn - 1
    low = 0
    norm = np.sum(np.abs(np.triu(H, -1)))
    ev = np.zeros(nn, dtype=complex)
    exshift = 0.0
    it = 0
    sweeps = slots = 0
    worst_order = 0.0
    while n >= low:
        l = low
        for cand in range(n, low, -1):
            sl = abs(H[cand - 1, cand - 1]) + abs(H[cand, cand])
            if sl == 0.0:
                sl = norm
            if abs(H[cand, cand - 1]) < EPS * sl:
                l = cand
                break
        x = H[n, n]
        if l == n:
            ev[n] = x + exshift
            n -= 1
            it = 0
            continue
        y = H[n - 1, n - 1]
        w = H[n, n - 1] * H[n - 1, n]
        if l == n - 1:
            p = (y - x) / 2.0
            q = p * p + w
            z = np.sqrt(abs(q))
            x += exshift
            if q >= 0:
                z = p + z if p >= 0 else p - z
                ev[n - 1] = x + z
                ev[n] = x - w / z if z != 0 else x + z
            else:
                ev[n - 1] = complex(x + p, z)
                ev[n] = complex(x + p, -z)
            n -= 2
            it = 0
            continue
        exc = it in (10, 30)
        if it == 10:
            exshift += x
            for i in range(low, n + 1):
                H[i, i] -= x
            s = abs(H[n, n - 1]) + abs(H[n - 1, n - 2])
            x = y = 0.75 * s
            w = -0.4375 * s * s
        if it == 30:
            s = (y - x) / 2.0
            s = s * s + w
            if s > 0:
                s = np.sqrt(s)
                if y < x:
                    s = -s
                s = x - w / ((y - x) / 2.0 + s)
                for i in range(low, n + 1):
                    H[i, i] -= s
                exshift += s
                x = y = w = 0.964
        it += 1
        if it > 60 * nn:
            raise RuntimeError("no convergence")
        # bulge start
        m = l
        for mm in range(n - 2, l - 1, -1):
            zz = H[mm, mm]
            r_, s_ = x - zz, y - zz
            p = (r_ * s_ - w) / H[mm + 1, mm] + H[mm, mm + 1]
            q = H[mm + 1, mm + 1] - zz - r_ - s_
            r = H[mm + 2, mm + 1]
            sc = abs(p) + abs(q) + abs(r)
            p, q, r = p / sc, q / sc, r / sc
            if mm == l:
                m = mm
                break
            if abs(H[mm, mm - 1]) * (abs(q) + abs(r)) < EPS * (abs(p) * (abs(H[mm - 1, mm - 1]) + abs(zz) + abs(H[mm + 1, mm + 1]))):
                m = mm
                break
        pqr = (p, q, r)
        sweeps += 1
        if two and not exc and m == l and n - l >= 5:
            # shifts of the 2 x 2 block above the trailing one, fixed before the sweep
            sh2 = (H[n - 2, n - 2], H[n - 3, n - 3], H[n - 2, n - 3] * H[n - 3, n - 2])
            if check_order:
                Hs = H.copy()
                sweep(Hs, l, n, m, pqr)
                sweep(Hs, l, n, l, intro(Hs, l, *sh2))
            slots += two_sweeps_pipelined(H, l, n, pqr, sh2)
            sweeps += 1
            if check_order:
                worst_order = max(worst_order, np.max(np.abs(np.triu(Hs - H, -1))) / norm)
        else:
            slots += sweep(H, l, n, m, pqr)
    return ev, sweeps, slots, worst_order


def ev_err(ev, A):
    ref = np.linalg.eigvals(A)
    used = np.zeros(len(ref), bool)
    worst = 0.0
    for v in ev:
        d = np.abs(ref - v)
        d[used] = np.inf
        j = int(np.argmin(d))
        used[j] = True
        worst = max(worst, d[j] / max(abs(ref[j]), 1e-300))
    return worst


def atilde(name):
    from oracle import cdmd as OD
    from oracle import sensing as OS
    from synth.scene import config_by_name, video_for
    cfg = config_by_name(name)
    X = video_for(cfg)
    kind = {"sparse": OS.SPARSE, "spixel": OS.SPIXEL, "rademacher": OS.RADEMACHER, "gaussian": OS.GAUSSIAN}[cfg.kind]
    Y = OS.sketch(X, kind, cfg.p, cfg.sensing_seed)
    return OD.fit(Y.astype(np.float64), cfg.k, cfg.K)["Atilde"]


def main():
    names = sys.argv[1:] or ["c2_320x240_spixel"]
    cases = []
    for nm in names:
        if nm.startswith("rand"):
            k = int(nm[4:] or 50)
            rng = np.random.default_rng(k)
            for t in range(3):
                cases.append((f"{nm}#{t}", rng.standard_normal((k, k))))
        else:
            cases.append((nm, atilde(nm)))
    for nm, A in cases:
        H0 = scipy.linalg.hessenberg(A)
        e1, sw1, sl1, _ = hqr(H0)
        e2, sw2, sl2, wo = hqr(H0, two=True, check_order=True)
        print(f"{nm:24s} k={A.shape[0]:3d}  one bulge: sweeps {sw1:4d} steps {sl1:5d} err {ev_err(e1, A):.1e}   "
              f"two bulges: sweeps {sw2:4d} slots {sl2:5d} err {ev_err(e2, A):.1e} order-vs-sequential {wo:.1e}")


if __name__ == "__main__":
    main()
