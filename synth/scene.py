"""Synthetic CDnet/HD-shaped grayscale videos (seeded, uint8, frame-major).

Recipe (shapes from BASELINE.json configs):
  x_t(j) = clamp(round( a(j)                                   smooth texture in [60, 180]
                      + b1(j) cos(pi (t-1) / 2) + b2(j) sin(pi (t-1) / 2)   period-4 pair, |b1|+|b2| <= 30
                      + f(j) (-1)^(t-1)                        optional period-2 flicker
                      + N(0, noise^2) ), 0, 255)
          overwritten by 1-3 moving rectangles of intensity 250 (side ~ h/5,
          1-4 px/frame, entering / leaving mid-batch, canoe-like).
The background terms are integer-valued, so with noise = 0 and no rectangles
the video is exactly periodic with period 4: its DMD eigenvalues are exactly
{1, i, -i} (the oracle pin of tests/test_oracle_dmd.py).

Every pixel slab [pix0, pix0 + n_local) can be generated on its own (noise is
drawn per (frame, 64-row block)), so each rank of a pixel-sharded run builds
exactly its own bytes of the same global video.
"""

from dataclasses import dataclass, field

import numpy as np

SPIXEL, SPARSE, RADEMACHER, GAUSSIAN = 0, 1, 2, 3
KIND = {"spixel": SPIXEL, "sparse": SPARSE, "rademacher": RADEMACHER, "gaussian": GAUSSIAN}
ROWBLK = 64


@dataclass(frozen=True)
class Config:
    name: str
    width: int
    height: int
    m: int
    kind: str
    p: int
    k: int
    K: int
    tau: float = 25.0
    noise: float = 2.0
    n_rects: int = 2
    flicker: bool = False
    video_seed: int = 1000
    sensing_seed: int = 0
    gpus: tuple = (1,)
    text: str = ""

    @property
    def n(self):
        return self.width * self.height


CONFIGS = [
    Config("c1_32x24_sparse", 32, 24, 40, "sparse", 50, 10, 2, noise=0.0, n_rects=1,
           video_seed=1001, gpus=(0,),
           text="synthetic 32x24, 40 frames, 3 Fourier background modes + moving square, sparse p=50, k=10, K=2"),
    Config("c2_320x240_spixel", 320, 240, 200, "spixel", 1000, 20, 10, video_seed=1002,
           text="CDnet-shaped 320x240, 200 frames, single-pixel p=1000, k=20"),
    Config("c3_720x480_rademacher", 720, 480, 300, "rademacher", 1500, 30, 10, video_seed=1003,
           gpus=(1, 2), text="720x480, 300 frames, Rademacher p=1500, k=30"),
    Config("c4_1080p_sparse", 1920, 1080, 500, "sparse", 2000, 50, 10, video_seed=1004,
           gpus=(1, 2, 4, 8), text="1920x1080 HD, 500 frames, sparse p=2000, k=50"),
    Config("c4_1080p_gaussian", 1920, 1080, 500, "gaussian", 2000, 50, 10, video_seed=1004,
           gpus=(1, 2, 4, 8), text="1920x1080 HD, 500 frames, Gaussian(bf16) p=2000, k=50"),
    Config("c5_4k_sparse", 3840, 2160, 1000, "sparse", 4000, 100, 10, video_seed=1005,
           gpus=(8,), text="3840x2160 4K, 1000 frames, sparse p=4000, k=100"),
]


def config_by_name(name):
    for c in CONFIGS:
        if c.name == name:
            return c
    raise KeyError(name)


def _smooth_field(rng, height, width, cell, lo, hi):
    """Bilinear upsampling of a coarse uniform grid -> smooth field in [lo, hi]."""
    gh, gw = height // cell + 2, width // cell + 2
    g = rng.uniform(lo, hi, size=(gh, gw))
    ys = np.arange(height) / cell
    xs = np.arange(width) / cell
    y0 = np.floor(ys).astype(int)
    x0 = np.floor(xs).astype(int)
    fy = (ys - y0)[:, None]
    fx = (xs - x0)[None, :]
    a = g[y0][:, x0] * (1 - fy) * (1 - fx) + g[y0 + 1][:, x0] * fy * (1 - fx) \
        + g[y0][:, x0 + 1] * (1 - fy) * fx + g[y0 + 1][:, x0 + 1] * fy * fx
    return a


@dataclass
class _Scene:
    a: np.ndarray
    b1: np.ndarray
    b2: np.ndarray
    f: np.ndarray
    rects: list = field(default_factory=list)


def _scene(cfg_w, cfg_h, m, seed, n_rects, flicker):
    rng = np.random.default_rng(seed)
    cell = max(4, min(cfg_w, cfg_h) // 6)
    a = np.rint(_smooth_field(rng, cfg_h, cfg_w, cell, 60, 180))
    r = _smooth_field(rng, cfg_h, cfg_w, cell, 0, 1)
    th = _smooth_field(rng, cfg_h, cfg_w, cell, 0, 2 * np.pi)
    amp = 30.0 * r / (np.abs(np.cos(th)) + np.abs(np.sin(th)))  # |b1| + |b2| <= 30
    b1 = np.trunc(amp * np.cos(th))
    b2 = np.trunc(amp * np.sin(th))
    f = np.trunc(_smooth_field(rng, cfg_h, cfg_w, cell, -8, 8)) if flicker else np.zeros_like(a)
    rects = []
    side = max(2, cfg_h // 5)
    for i in range(n_rects):
        speed = rng.uniform(1, 4)
        ang = rng.uniform(-0.4, 0.4) + (0 if i % 2 == 0 else np.pi)
        vx, vy = speed * np.cos(ang), speed * np.sin(ang)
        # start so that the rectangle crosses the frame around the middle of the batch
        cx = cfg_w / 2 - vx * m / 2 + rng.uniform(-cfg_w / 6, cfg_w / 6)
        cy = cfg_h / 2 - vy * m / 2 + rng.uniform(-cfg_h / 6, cfg_h / 6)
        w = int(max(2, side * rng.uniform(0.8, 1.6)))
        h = int(max(2, side * rng.uniform(0.8, 1.2)))
        rects.append((cx, cy, vx, vy, w, h))
    return _Scene(a, b1, b2, f, rects)


def make_video(width, height, m, seed, noise=2.0, n_rects=2, flicker=False,
               pix0=0, n_local=None, periodic=True, threads=None):
    """Return uint8 array (m, n_local): frame t holds global pixels [pix0, pix0+n_local)."""
    from concurrent.futures import ThreadPoolExecutor
    import os

    n = width * height
    n_local = n - pix0 if n_local is None else n_local
    sc = _scene(width, height, m, seed, n_rects, flicker)
    r0 = pix0 // width
    r1 = (pix0 + n_local + width - 1) // width
    b0 = r0 // ROWBLK
    b1_ = (r1 + ROWBLK - 1) // ROWBLK
    R0, R1 = b0 * ROWBLK, min(height, b1_ * ROWBLK)
    a = sc.a[R0:R1]
    z = np.zeros_like(a)
    pb1 = sc.b1[R0:R1] if periodic else z
    pb2 = sc.b2[R0:R1] if periodic else z
    ff = sc.f[R0:R1]
    cos4 = [1, 0, -1, 0]
    sin4 = [0, 1, 0, -1]
    # the four (eight with flicker) distinct noiseless background frames
    base = {}
    for ph in range(4):
        for fl in (0, 1):
            base[(ph, fl)] = (a + cos4[ph] * pb1 + sin4[ph] * pb2 + (1 - 2 * fl) * ff).astype(np.float32)
    out = np.empty((m, n_local), dtype=np.uint8)
    off = pix0 - R0 * width

    def frame(t):
        fr = base[(t % 4, t % 2)].copy()
        if noise > 0:
            for b in range(b0, b1_):
                lo, hi = b * ROWBLK - R0, min(R1, (b + 1) * ROWBLK) - R0
                g = np.random.default_rng([seed, 7, t, b])
                fr[lo:hi] += g.standard_normal((hi - lo, width), dtype=np.float32) * np.float32(noise)
        for (cx, cy, vx, vy, w, h) in sc.rects:
            x0 = int(round(cx + vx * t - w / 2))
            y0 = int(round(cy + vy * t - h / 2))
            xa, xb = max(0, x0), min(width, x0 + w)
            ya, yb = max(R0, y0), min(R1, y0 + h)
            if xa < xb and ya < yb:
                fr[ya - R0:yb - R0, xa:xb] = 250.0
        np.rint(fr, out=fr)
        np.clip(fr, 0, 255, out=fr)
        out[t] = fr.reshape(-1)[off:off + n_local].astype(np.uint8)

    nthreads = threads or min(16, os.cpu_count() or 1)
    if m * n_local < (1 << 20) or nthreads == 1:
        for t in range(m):
            frame(t)
    else:
        with ThreadPoolExecutor(nthreads) as ex:
            list(ex.map(frame, range(m)))
    return out


def video_for(cfg, pix0=0, n_local=None):
    return make_video(cfg.width, cfg.height, cfg.m, cfg.video_seed, noise=cfg.noise,
                      n_rects=cfg.n_rects, flicker=cfg.flicker, pix0=pix0, n_local=n_local)
