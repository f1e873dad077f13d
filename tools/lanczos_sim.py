"""Lanczos step-count study for lanczos.cu (host-side NumPy, not on the product path).

Builds the snapshot Gram Y^T Y of a config's sketch, runs Lanczos with two-pass classical
Gram-Schmidt exactly as lz_kernel orders it, and prints, per Krylov dimension J, the
worst residual-over-gap ratio |beta_{J-1} s_{J-1,i}| / (theta_i - theta_k) of the k
largest Ritz pairs (the convergence test lz_check_kernel applies, threshold 1e-9) and
the worst Ritz-vector error against numpy.linalg.eigh.
usage: python tools/lanczos_sim.py c4 [c1 ...]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from synth.scene import config_by_name, video_for  # noqa: E402
from oracle import sensing as OS  # noqa: E402


def lanczos(G, J, rng):
    n = G.shape[0]
    Q = np.zeros((n, J))
    q = rng.uniform(-0.5, 0.5, n)
    Q[:, 0] = q / np.linalg.norm(q)
    al, be = np.zeros(J), np.zeros(J)
    for j in range(J):
        z = G @ Q[:, j]
        h1 = Q[:, : j + 1].T @ z
        z = z - Q[:, : j + 1] @ h1
        nz1 = z @ z
        h2 = Q[:, : j + 1].T @ z
        z = z - Q[:, : j + 1] @ h2
        al[j] = h1[j] + h2[j]
        be[j] = np.sqrt(max(nz1 - h2 @ h2, 0.0))
        if j + 1 < J:
            Q[:, j + 1] = z / be[j]
    return Q, al, be


def main():
    for name in sys.argv[1:]:
        cfg = config_by_name(name)
        X = video_for(cfg)
        Y = OS.sketch(X, {"sparse": OS.SPARSE, "spixel": OS.SPIXEL}.get(cfg.kind, OS.SPARSE), cfg.p, cfg.sensing_seed)
        Y = Y.astype(np.float64)[:, :-1]
        G = Y.T @ Y
        k = cfg.k
        w, U = np.linalg.eigh(G)
        print(f"{name}: n={G.shape[0]} k={k} lam_k/lam_k+1={w[-k] / w[-k - 1]:.4f}")
        for J in range(2 * k, min(G.shape[0], 3 * k + 20), 5):
            Q, al, be = lanczos(G, J, np.random.default_rng(1))
            T = np.diag(al) + np.diag(be[:-1], 1) + np.diag(be[:-1], -1)
            th, S = np.linalg.eigh(T)
            th, S = th[-k - 1:], S[:, -k - 1:]
            ratio = max(abs(be[-1] * S[-1, q]) / (th[q] - th[0]) for q in range(1, k + 1))
            V = Q @ S[:, 1:]
            err = 0.0
            for q in range(k):
                u = U[:, -k + q]
                err = max(err, np.linalg.norm(V[:, q] - np.sign(u @ V[:, q]) * u))
            lerr = np.max(np.abs(th[1:] - w[-k:]) / w[-k:])
            print(f"  J={J:4d} resid/gap={ratio:.2e} vec_err={err:.2e} eig_relerr={lerr:.2e}")


if __name__ == "__main__":
    main()
