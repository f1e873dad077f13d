"""Fan the oracle's own per-pixel steps over pixel slabs in worker processes.

TEST INFRASTRUCTURE — see oracle/__init__.py.  This module holds no arithmetic of
the method: every number comes from oracle.cdmd.modes / background_dynamic /
background_static / mask (and oracle.sensing.sketch), called unchanged on column
slabs of the video.  Those steps are per pixel ("embarrassingly parallel"),
so the slab results concatenate to the whole-frame results bit for bit.  It exists so
the full-frame oracle fits the test / bench time budget on a many-core host.

Each worker generates its own slab of the seeded synthetic video once
(synth.video_for(cfg, pix0, n_local): the same bytes as the whole video's columns)
and keeps it for every call.

    with PixelPool(cfg, workers=16) as pool:
        out = pool.run(model, tau, dynamic=True, want=("Phi", "mask", "band"))
"""

import multiprocessing as mp
import os

import numpy as np


def _worker(conn, cfg_name, pix0, n_local):
    from synth.scene import config_by_name, video_for
    from . import cdmd as OD
    cfg = config_by_name(cfg_name)
    X = video_for(cfg, pix0=pix0, n_local=n_local)
    conn.send(("ready", pix0, n_local))
    while True:
        msg = conn.recv()
        if msg is None:
            break
        model, tau, dynamic, want, chunk = msg
        res = {k: [] for k in want}
        npos = 0
        for c0 in range(0, n_local, chunk):
            c1 = min(n_local, c0 + chunk)
            Xc = X[:, c0:c1]
            Phi = OD.modes(Xc, model["M"])
            L = OD.background_dynamic(Phi, model) if dynamic else OD.background_static(Phi, model)
            Mk = OD.mask(Xc, L, tau)
            npos += int(Mk.sum())
            if "Phi" in res:
                res["Phi"].append(Phi)
            if "mask" in res:
                res["mask"].append(Mk)
            if "band" in res:   # pixels whose oracle residual lies within 1e-3 of tau
                Lt = L[None, :] if L.ndim == 1 else L.T
                res["band"].append(np.abs(np.abs(Xc.astype(np.float64) - Lt) - tau) <= 1e-3)
        out = {k: np.concatenate(v, axis=1 if k in ("mask", "band") else 0) for k, v in res.items() if v}
        for k in ("mask", "band"):   # bit-packed for the trip through the pipe
            if k in out:
                out[k] = np.packbits(out[k], axis=1, bitorder="little")
        out["count"] = npos
        conn.send(out)
    conn.close()


def _slabs(n, parts):
    b = [(n * i) // parts for i in range(parts + 1)]
    return [(b[i], b[i + 1] - b[i]) for i in range(parts) if b[i + 1] > b[i]]


def _slab_sketch(cfg_name, kind, pix0, nl):
    from synth.scene import config_by_name, video_for
    from . import sensing as OS
    cfg = config_by_name(cfg_name)
    Xs = video_for(cfg, pix0=pix0, n_local=nl)
    return OS.sketch(Xs, kind, cfg.p, cfg.sensing_seed, n_total=cfg.n, pix0=pix0, chunk=1 << 14)


def parallel_sketch(cfg, kind, workers=None):
    """Y_full = C D of cfg's video as the sum of the oracle's per-slab partial sketches
    (columns of C indexed by the global pixel, so slabs sum to the whole sketch; pinned
    by tests/test_oracle_sensing.py), the slabs computed in worker processes."""
    nw = workers or max(1, min(32, len(os.sched_getaffinity(0))))
    parts = _slabs(cfg.n, nw)
    with _single_thread_blas():
        with mp.get_context("spawn").Pool(len(parts)) as pool:
            ys = pool.starmap(_slab_sketch, [(cfg.name, kind, p0, nl) for p0, nl in parts])
    return np.sum(ys, axis=0)


class _single_thread_blas:
    """One BLAS thread per worker (the workers already use every core); spawned
    interpreters inherit the environment at spawn time."""

    def __enter__(self):
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        env = {"PYTHONPATH": root + (os.pathsep + os.environ["PYTHONPATH"] if os.environ.get("PYTHONPATH") else ""),
               "OMP_NUM_THREADS": "1", "OPENBLAS_NUM_THREADS": "1", "MKL_NUM_THREADS": "1"}
        self.saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        return self

    def __exit__(self, *a):
        for k, v in self.saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


class PixelPool:
    """Worker processes, each owning a contiguous pixel slab of cfg's video."""

    def __init__(self, cfg, workers=None, chunk=1 << 15):
        ctx = mp.get_context("spawn")
        nw = workers or max(1, min(32, len(os.sched_getaffinity(0))))
        self.cfg, self.chunk = cfg, chunk
        self.parts = _slabs(cfg.n, nw)
        self.conns, self.procs = [], []
        with _single_thread_blas():
            for pix0, nl in self.parts:
                a, b = ctx.Pipe()
                p = ctx.Process(target=_worker, args=(b, cfg.name, pix0, nl), daemon=True)
                p.start()
                self.conns.append(a)
                self.procs.append(p)
        for c in self.conns:
            assert c.recv()[0] == "ready"
        self.cores = len(self.parts)

    def run(self, model, tau, dynamic=True, want=()):
        """Modes, background and mask of every pixel, slab by slab in parallel.
        Returns dict: "count" (foreground pixels), and per `want`: "Phi" (n x k
        complex128), "mask" (m x n bool), "band" (m x n bool: |res - tau| <= 1e-3)."""
        keep = ("M", "lam", "beta", "support", "m")
        small = {k: model[k] for k in keep}
        for c in self.conns:
            c.send((small, tau, dynamic, tuple(want), self.chunk))
        outs = [c.recv() for c in self.conns]
        res = {"count": sum(o["count"] for o in outs)}
        for k in want:
            if k in ("mask", "band"):
                res[k] = np.concatenate([np.unpackbits(o[k], axis=1, count=nl, bitorder="little").astype(bool)
                                         for o, (_, nl) in zip(outs, self.parts)], axis=1)
            else:
                res[k] = np.concatenate([o[k] for o in outs], axis=0)
        return res

    def close(self):
        for c in self.conns:
            try:
                c.send(None)
            except Exception:
                pass
        for p in self.procs:
            p.join(timeout=30)
            if p.is_alive():
                p.terminate()
        self.conns, self.procs = [], []

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
